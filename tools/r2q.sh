timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_resnet.py -q -x > gpurun_out/r2q_tests.log 2>&1; echo rc=$? >> gpurun_out/r2q_tests.log
for L in layer1.0.conv3 conv1; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2q_launches_$L.csv python tools/one_layer.py $L 2 > /dev/null 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2q_launches_c2.csv python tools/one_step.py --config c2 --steps 2 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_fused_small -c 1 -o gpurun_out/r2q_fs python tools/one_layer.py layer1.0.conv3 1 > /dev/null 2>&1
