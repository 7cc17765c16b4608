# K8w (128 x 256 tiles, TC correction): guarded parity run, then A/B vs K8 at c2 / c4
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -q -x > gpurun_out/r5p_tests.log 2>&1; echo rc=$? >> gpurun_out/r5p_tests.log
if grep -q "rc=0" gpurun_out/r5p_tests.log; then
  for W in 1 0; do
    LRQMM_K8W=$W timeout 300 python bench.py --config c2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r5p_c2_w$W.json 2>&1
    LRQMM_K8W=$W timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k8 --csv --log-file gpurun_out/r5p_k8_c2_w$W.csv python tools/one_step.py --config c2 --steps 2 > /dev/null 2>&1
    LRQMM_K8W=$W timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r5p_c4_w$W.json 2>&1
  done
  timeout 600 python -m pytest tests/test_gpu_resnet.py tests/test_gpu_multirank.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r5p_tests2.log 2>&1; echo rc=$? >> gpurun_out/r5p_tests2.log
fi
