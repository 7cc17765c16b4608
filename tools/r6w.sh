# one CholQR fused_small launch (layer4.2.conv3), full set with source
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fused_small" --launch-skip 1 -c 1 -o gpurun_out/r6w_fs python tools/one_layer.py layer4.2.conv3 1 > gpurun_out/r6w.log 2>&1
