# shared-space smem base in the TMA/UMMA kernels (was generic LD/ST in the epilogues)
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r6x_tests.log 2>&1; echo rc=$? >> gpurun_out/r6x_tests.log
for c in c2 c3; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r6x_bench_$c.json 2>&1; done
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r6x_bench_c4.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r6x_l1.csv python tools/one_layer.py layer1.0.conv3 2 > /dev/null 2>&1
