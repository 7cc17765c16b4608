# CholQR: batched G loads, G staged in shared memory by the fused Gram kernel
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x > gpurun_out/r3x_tests.log 2>&1; echo rc=$? >> gpurun_out/r3x_tests.log
for c in c2 c3; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r3x_bench_$c.json 2>&1; done
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r3x_bench_c4.json 2>&1
timeout 2000 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3x_c4_all.csv python tools/c4_all.py > gpurun_out/r3x_c4.log 2>&1
