ncu --set full --import-source on --clock-control none -k regex:k_fused_small -s 1 -c 1 -o gpurun_out/r2p_fs python tools/one_layer.py layer1.0.conv3 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_apply64 -c 1 -o gpurun_out/r2p_ap python tools/one_layer.py layer1.0.conv3 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_apply_small -c 1 -o gpurun_out/r2p_as python tools/one_layer.py layer1.0.conv3 1 > /dev/null 2>&1
