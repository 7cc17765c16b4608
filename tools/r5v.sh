# Gram with a one-column tail block on FP64 FMAs (6 instead of 10 DMMAs per slice at 25 of 32 columns)
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_resnet.py -q -x > gpurun_out/r5v_tests.log 2>&1; echo rc=$? >> gpurun_out/r5v_tests.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_fused_small --csv --log-file gpurun_out/r5v_fs.csv python tools/one_layer.py layer1.0.conv3 2 > /dev/null 2>&1
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r5v_bench_c4.json 2>&1
