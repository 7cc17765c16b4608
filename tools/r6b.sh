# im2col tile: 16 lanes x 9 quads for 3x3 / C = 64 rows
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "im2col" tests/test_gpu_resnet.py > gpurun_out/r6b_tests.log 2>&1; echo rc=$? >> gpurun_out/r6b_tests.log
for V in 1 0; do
  LRQMM_IM2COL_L16=$V timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:im2col --csv --log-file gpurun_out/r6b_l1_$V.csv python tools/one_layer.py layer1.0.conv2 2 > /dev/null 2>&1
done
