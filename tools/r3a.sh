timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r3a_gpu.log 2>&1; echo rc=$? >> gpurun_out/r3a_gpu.log
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 > gpurun_out/r3a_bench_c4.json 2>&1
timeout 300 python bench.py --config c2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r3a_bench_c2.json 2>&1
