# short-row K1 (rows_tma): lanes per row sweep on c4 1x1 layers; parity
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "quantize" > gpurun_out/r3z_tests.log 2>&1; echo rc=$? >> gpurun_out/r3z_tests.log
for L in layer1.0.conv1 layer1.1.conv1 layer2.0.conv3 layer3.0.conv1 layer4.0.conv1; do
  for F in 1 2 4 8; do
    LRQMM_K1_F4PL=$F timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rows_tma --csv --log-file gpurun_out/r3z_${L}_$F.csv python tools/one_layer.py $L 3 > /dev/null 2>&1
  done
done
