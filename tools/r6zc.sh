# apply64_tc: per-slab outputs, 4 blocks per SM
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r6zc_tests.log 2>&1; echo rc=$? >> gpurun_out/r6zc_tests.log
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r6zc_bench_c4.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_shared_mem --clock-control none -k regex:"k_assemble|k_apply64_tc" --csv --log-file gpurun_out/r6zc_asm.csv python tools/one_layer.py layer1.0.conv3 2 > /dev/null 2>&1
