timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2h_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2h_gpu.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2h_launches_c2.csv python tools/one_step.py --config c2 --steps 3 > gpurun_out/r2h_ncu_c2.log 2>&1
timeout 300 python bench.py --config c2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2h_bench_c2.json 2>&1
LRQMM_RSVD_LEGACY=1 timeout 300 python bench.py --config c2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2h_bench_c2_legacy.json 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2h_bench_c3.json 2>&1
