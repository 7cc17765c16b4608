# K8 GEMM on output-heavy c4 layers: ncu full
for L in layer1.0.conv3 layer1.0.conv1; do
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k8_gemm -s 1 -c 1 -o gpurun_out/r4a_k8_$L python tools/one_layer.py $L 2 > /dev/null 2>&1
done
