timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2z_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2z_gpu.log
timeout 2000 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2z_c4_all.csv python tools/c4_all.py > gpurun_out/r2z_c4.log 2>&1
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 > gpurun_out/r2z_bench_c4.json 2>&1
