# S3: one reduction launch for both dual-pass outputs
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x > gpurun_out/r5e_tests.log 2>&1; echo rc=$? >> gpurun_out/r5e_tests.log
for c in c2 c3; do timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r5e_bench_$c.json 2>&1; done
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r5e_bench_c4.json 2>&1
