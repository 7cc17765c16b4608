timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_chain or lrqmm_matches or static_b or deterministic or rank_and_power" > gpurun_out/r2e_tests.log 2>&1; echo rc=$? >> gpurun_out/r2e_tests.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2e_launches_c2.csv python tools/one_step.py --config c2 --steps 3 > gpurun_out/r2e_ncu_c2.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2e_launches_c3.csv python tools/one_step.py --config c3 --steps 2 > gpurun_out/r2e_ncu_c3.log 2>&1
timeout 300 python bench.py --config c2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2e_bench_c2.json 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2e_bench_c3.json 2>&1
