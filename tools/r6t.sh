# k_assemble profile (layer1.0.conv3)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_assemble" -c 1 -o gpurun_out/r6t_asm python tools/one_layer.py layer1.0.conv3 1 > gpurun_out/r6t.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "widest" > gpurun_out/r6t_tests.log 2>&1; echo rc=$? >> gpurun_out/r6t_tests.log
