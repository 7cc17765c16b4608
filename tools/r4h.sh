# evidence refresh: full GPU tests, smoke, bench lines (c3 default with cpu_baseline + e2e, c2, c4, c5), reference arm, c3 launch list
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r4h_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r4h_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r4h_smoke.log 2>&1; echo rc=$? >> gpurun_out/r4h_smoke.log
timeout 900 python bench.py > gpurun_out/r4h_bench_c3.json 2> gpurun_out/r4h_bench_c3.err
timeout 600 python bench.py --config c2 --steps 50 --warmup 5 > gpurun_out/r4h_bench_c2.json 2> gpurun_out/r4h_bench_c2.err
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/r4h_bench_c4.json 2> gpurun_out/r4h_bench_c4.err
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r4h_bench_c5.json 2> gpurun_out/r4h_bench_c5.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r4h_bench_ref.json 2> gpurun_out/r4h_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r4h_launches_c3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r4h_ncu_c3.log 2>&1
