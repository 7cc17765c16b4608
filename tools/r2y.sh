timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2y_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2y_gpu.log
timeout 300 python bench.py --config c2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2y_bench_c2.json 2>&1
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 > gpurun_out/r2y_bench_c4.json 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2y_bench_c3.json 2>&1
