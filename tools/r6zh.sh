# row K1 (short rows) chunk / slot sweep on K = 64 / 256 / 512 layers
for L in layer1.0.conv3 layer1.1.conv1 layer2.1.conv1; do
 for cfg in "8192 3" "8192 4" "16384 3" "4096 4" "4096 6"; do
  set -- $cfg
  LRQMM_K1R_CHUNK=$1 LRQMM_K1R_SLOTS=$2 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k1_quantize_rows --csv --log-file gpurun_out/r6zh_${L}_$1_$2.csv python tools/one_layer.py $L 2 > /dev/null 2>&1
  echo "$L chunk=$1 slots=$2: $(grep -h gpu__time_duration gpurun_out/r6zh_${L}_$1_$2.csv | awk -F'","' '{gsub(/"/,"",$NF); printf "%.1f ", $NF/1000}')" >> gpurun_out/r6zh.log
 done
done
