timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_resnet.py tests/test_gpu_multirank.py -q -x > gpurun_out/r2s_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s_tests.log
for L in layer1.0.conv3 conv1; do
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s_launches_$L.csv python tools/one_layer.py $L 2 > /dev/null 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s_launches_c2.csv python tools/one_step.py --config c2 --steps 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s_launches_c3.csv python tools/one_step.py --config c3 --steps 2 > /dev/null 2>&1
