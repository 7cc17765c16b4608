# K8 / K8w epilogue: next chunk's TMEM loads issued before this chunk's stores
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_resnet.py -q -x > gpurun_out/r5z_tests.log 2>&1; echo rc=$? >> gpurun_out/r5z_tests.log
for L in layer1.0.conv3 layer1.0.conv1 layer3.0.conv3 layer4.0.conv2; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k8 --csv --log-file gpurun_out/r5z_k8_$L.csv python tools/one_layer.py $L 2 > /dev/null 2>&1
done
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r5z_bench_c4.json 2>&1
timeout 600 python bench.py --config c2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r5z_bench_c2.json 2>&1
