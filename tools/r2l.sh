timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2l_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2l_gpu.log
timeout 300 python bench.py --config c2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2l_bench_c2.json 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2l_bench_c3.json 2> gpurun_out/r2l_bench_c3.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2l_launches_c3.csv python tools/one_step.py --config c3 --steps 2 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k7_gemm -s 1 -c 1 -o gpurun_out/r2l_gemm_c3 python tools/one_step.py --config c3 --steps 2 > /dev/null 2>&1
