timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2i_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2i_gpu.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2i_launches_c2.csv python tools/one_step.py --config c2 --steps 3 > gpurun_out/r2i_ncu_c2.log 2>&1
for w in 3 2 1; do LRQMM_TC_WAVES=$w timeout 300 python bench.py --config c2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2i_bench_c2_w$w.json 2>&1; done
for w in 3 2; do LRQMM_TC_WAVES=$w timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2i_bench_c3_w$w.json 2>&1; done
