# K8 epilogue with the warp-private smem transpose: parity, per-layer GEMM time, benches
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_resnet.py -q -x > gpurun_out/r4b_tests.log 2>&1; echo rc=$? >> gpurun_out/r4b_tests.log
for L in layer1.0.conv3 layer1.0.conv1 layer3.0.conv3 layer4.0.conv3; do
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k8_gemm --csv --log-file gpurun_out/r4b_k8_$L.csv python tools/one_layer.py $L 3 > /dev/null 2>&1
done
for c in c2 c3; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r4b_bench_$c.json 2>&1; done
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r4b_bench_c4.json 2>&1
