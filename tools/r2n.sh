for K in k_fused_small k_apply64 k_apply_small k6_gemm; do
ncu --set full --import-source on --clock-control none -k regex:$K -s 2 -c 1 -o gpurun_out/r2n_$K python tools/one_layer.py layer1.0.conv3 2 > /dev/null 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:k1_quantize_im2col -c 1 -o gpurun_out/r2n_im2col_conv1 python tools/one_layer.py conv1 1 > /dev/null 2>&1
