# tiled implicit im2col: parity, per-layer K1 time (tile vs gather), c4 bench, one ncu capture
timeout 900 python -m pytest tests/test_gpu_parity.py -k "im2col" tests/test_gpu_resnet.py -q -x > gpurun_out/r3f_tests.log 2>&1; echo rc=$? >> gpurun_out/r3f_tests.log
for L in conv1 layer1.0.conv2 layer2.0.conv2 layer3.1.conv2 layer4.0.conv2; do
  for V in tile gather; do
    if [ $V = gather ]; then export LRQMM_IM2COL_GATHER=1; else unset LRQMM_IM2COL_GATHER; fi
    timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:im2col --csv --log-file gpurun_out/r3f_${L}_$V.csv python tools/one_layer.py $L 3 > /dev/null 2>&1
  done
done
unset LRQMM_IM2COL_GATHER
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r3f_bench_c4.json 2>&1
LRQMM_IM2COL_GATHER=1 timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r3f_bench_c4_gather.json 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:im2col -c 1 -o gpurun_out/r3f_im2col_conv1 python tools/one_layer.py conv1 1 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:im2col -c 1 -o gpurun_out/r3f_im2col_l1c2 python tools/one_layer.py layer1.0.conv2 1 > /dev/null 2>&1
