# CholQR: batched G loads, G staged in shared memory by the fused Gram kernel
./tools/eig_bench > gpurun_out/r3l_eig.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x > gpurun_out/r3l_tests.log 2>&1; echo rc=$? >> gpurun_out/r3l_tests.log
for c in c2 c3; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r3l_bench_$c.json 2>&1; done
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r3l_bench_c4.json 2>&1
