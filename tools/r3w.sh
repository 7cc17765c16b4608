# c4 per-kernel breakdown (current build) + apply kernels on a tall layer
timeout 2000 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3w_c4_all.csv python tools/c4_all.py > gpurun_out/r3w_c4.log 2>&1
for K in k_apply_small k_apply64 k_split_bf16 k_prep_img; do
timeout 300 ncu --set full --import-source on --clock-control none -k regex:$K -c 1 -o gpurun_out/r3w_$K python tools/one_layer.py layer1.0.conv3 2 > /dev/null 2>&1
done
