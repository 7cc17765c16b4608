# passes: a stage slot keeps its B image across units (no re-copy of the same image)
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_resnet.py -q -x > gpurun_out/r5t_tests.log 2>&1; echo rc=$? >> gpurun_out/r5t_tests.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_tc_proj --csv --log-file gpurun_out/r5t_proj.csv python tools/one_layer.py layer1.0.conv3 2 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_tc_proj --csv --log-file gpurun_out/r5t_proj_l3.csv python tools/one_layer.py layer3.1.conv1 2 > /dev/null 2>&1
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r5t_bench_c4.json 2>&1
for c in c2 c3; do timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r5t_bench_$c.json 2>&1; done
