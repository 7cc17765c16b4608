# pass epilogue: paired TMEM loads, transposed stores for the non-dual passes
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x > gpurun_out/r4g_tests.log 2>&1; echo rc=$? >> gpurun_out/r4g_tests.log
for L in layer1.0.conv3 layer2.0.conv2; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_tc_proj --csv --log-file gpurun_out/r4g_proj_$L.csv python tools/one_layer.py $L 2 > /dev/null 2>&1
done
for c in c2 c3; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r4g_bench_$c.json 2>&1; done
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r4g_bench_c4.json 2>&1
