# K8w vs K8 per c4 layer (N >= 256): GEMM time
for L in layer1.0.conv3 layer2.0.conv3 layer3.0.conv1 layer3.0.conv2 layer3.0.conv3 layer4.0.conv1 layer4.0.conv2 layer4.0.conv3; do
  for W in 2 0; do
    LRQMM_K8W=$W timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k8 --csv --log-file gpurun_out/r5q_${L}_w$W.csv python tools/one_layer.py $L 2 > /dev/null 2>&1
  done
done
