# split-K partials summed inside the fused Gram kernel: parity (incl. fused-chain equality), benches
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r4n_tests.log 2>&1; echo rc=$? >> gpurun_out/r4n_tests.log
for c in c2 c3; do timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r4n_bench_$c.json 2>&1; done
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r4n_bench_c4.json 2>&1
