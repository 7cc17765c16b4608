# assembly of tall single-input jobs: direct loads (no staging) vs staged
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_resnet.py -q -x > gpurun_out/r5g_tests.log 2>&1; echo rc=$? >> gpurun_out/r5g_tests.log
for D in 1 0; do
LRQMM_APPLY_DIRECT=$D timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:apply_ --csv --log-file gpurun_out/r5g_apply_d$D.csv python tools/one_layer.py layer1.0.conv3 2 > /dev/null 2>&1
LRQMM_APPLY_DIRECT=$D timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r5g_bench_c4_d$D.json 2>&1
done
