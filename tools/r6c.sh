# im2col tile: 32 lanes x 9 quads for 3x3 / C = 128 rows (one register batch)
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "im2col" tests/test_gpu_resnet.py > gpurun_out/r6c_tests.log 2>&1; echo rc=$? >> gpurun_out/r6c_tests.log
for V in 1 0; do
  LRQMM_IM2COL_L16=$V timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:im2col --csv --log-file gpurun_out/r6c_l2_$V.csv python tools/one_layer.py layer2.1.conv2 2 > /dev/null 2>&1
done
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r6c_bench_c4.json 2>&1
