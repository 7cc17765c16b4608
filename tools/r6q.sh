# ncu --set full of the tall-panel kernels of layer1.0.conv3 (M = 802816, K = 64): apply_small, apply64_tc, fused_small, split
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_apply_small|k_apply64_tc|k_fused_small|k_split_bf16|k_prep_img" -c 12 -o gpurun_out/r6q_tall python tools/one_layer.py layer1.0.conv3 1 > gpurun_out/r6q.log 2>&1
