timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -q -x > gpurun_out/r3b_tests.log 2>&1; echo rc=$? >> gpurun_out/r3b_tests.log
for c in c3 c2; do
timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r3b_bench_$c.json 2>&1
LRQMM_RSVD_ONE_STREAM=1 timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r3b_bench_${c}_one.json 2>&1
done
