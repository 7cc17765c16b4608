# evidence refresh 5 (session 3 final build): full GPU tests, smoke, bench lines, reference arm, c3 launch list of one full call
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r6zo_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r6zo_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r6zo_smoke.log 2>&1; echo rc=$? >> gpurun_out/r6zo_smoke.log
timeout 900 python bench.py > gpurun_out/r6zo_bench_c3.json 2> gpurun_out/r6zo_bench_c3.err
timeout 600 python bench.py --config c2 --steps 50 --warmup 5 > gpurun_out/r6zo_bench_c2.json 2> gpurun_out/r6zo_bench_c2.err
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/r6zo_bench_c4.json 2> gpurun_out/r6zo_bench_c4.err
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r6zo_bench_c5.json 2> gpurun_out/r6zo_bench_c5.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r6zo_bench_ref.json 2> gpurun_out/r6zo_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r6zo_launches_c3.csv python tools/one_step.py --config c3 --steps 2 > gpurun_out/r6zo_ncu_c3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r6zo_launches_c2.csv python tools/one_step.py --config c2 --steps 3 > gpurun_out/r6zo_ncu_c2.log 2>&1
