# tiled implicit im2col v3 (cp.async double buffer, sub-warp rows): parity, per-layer K1 time sweep, c4 bench
timeout 900 python -m pytest tests/test_gpu_parity.py -k "im2col" tests/test_gpu_resnet.py -q -x > gpurun_out/r3g_tests.log 2>&1; echo rc=$? >> gpurun_out/r3g_tests.log
for L in conv1 layer1.0.conv2 layer2.0.conv2 layer2.1.conv2 layer3.0.conv2 layer3.1.conv2 layer4.0.conv2 layer4.1.conv2 layer2.0.downsample; do
  for V in 56_8 100_8 32_8 56_4 gather; do
    if [ $V = gather ]; then export LRQMM_IM2COL_GATHER=1; else unset LRQMM_IM2COL_GATHER; export LRQMM_IM2COL_SMEM_KB=${V%_*} LRQMM_IM2COL_MIN_TW=${V#*_}; fi
    timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:im2col --csv --log-file gpurun_out/r3g_${L}_$V.csv python tools/one_layer.py $L 3 > /dev/null 2>&1
  done
done
unset LRQMM_IM2COL_GATHER LRQMM_IM2COL_SMEM_KB LRQMM_IM2COL_MIN_TW
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r3g_bench_c4.json 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:im2col -c 1 -o gpurun_out/r3g_im2col_conv1 python tools/one_layer.py conv1 1 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:im2col -c 1 -o gpurun_out/r3g_im2col_l1c2 python tools/one_layer.py layer1.0.conv2 1 > /dev/null 2>&1
