# apply64 on the fp64 tensor cores (DMMA) vs the FMA form: parity, per-layer time, benches
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x > gpurun_out/r4l_tests.log 2>&1; echo rc=$? >> gpurun_out/r4l_tests.log
for V in tc fma; do
  if [ $V = fma ]; then export LRQMM_APPLY_FMA=1; else unset LRQMM_APPLY_FMA; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_apply_small --csv --log-file gpurun_out/r4l_apply_$V.csv python tools/one_layer.py layer1.0.conv3 2 > /dev/null 2>&1
  for c in c2 c3; do timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r4l_bench_${c}_$V.json 2>&1; done
  timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r4l_bench_c4_$V.json 2>&1
done
