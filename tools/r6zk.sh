# K8 vs K8w at narrow N / short K (c4 layers), and the c4 suite with K8w everywhere
for L in layer1.0.conv3 layer1.1.conv1 layer2.0.conv3 layer3.0.conv3; do
 for w in 1 2; do
  LRQMM_K8W=$w timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k8" --csv --log-file gpurun_out/r6zk_${L}_$w.csv python tools/one_layer.py $L 2 > /dev/null 2>&1
  echo "$L K8W=$w: $(grep -h gpu__time_duration gpurun_out/r6zk_${L}_$w.csv | awk -F'","' '{gsub(/"/,"",$NF); printf "%.1f ", $NF/1000}')" >> gpurun_out/r6zk.log
 done
done
LRQMM_K8W=2 timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r6zk_bench_c4_w2.json 2>&1
