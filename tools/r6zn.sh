# deep-window fallback of the tiled im2col: tests + c4
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r6zn_tests.log 2>&1; echo rc=$? >> gpurun_out/r6zn_tests.log
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r6zn_bench_c4.json 2>&1
