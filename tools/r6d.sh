# gather im2col: batch size by row length
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "im2col" tests/test_gpu_resnet.py > gpurun_out/r6d_tests.log 2>&1; echo rc=$? >> gpurun_out/r6d_tests.log
for L in layer2.0.conv2 layer3.1.conv2 layer4.1.conv2 layer2.0.downsample layer3.0.downsample; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:im2col --csv --log-file gpurun_out/r6d_$L.csv python tools/one_layer.py $L 2 > /dev/null 2>&1
done
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r6d_bench_c4.json 2>&1
