# tiled im2col for C >= 256 (larger smem budget / narrower tiles) vs the gather kernel
for L in layer3.1.conv2 layer4.1.conv2 layer3.0.conv2 layer2.0.conv2; do
 for cfg in "56 8" "100 7" "100 4" "80 4"; do
  set -- $cfg
  LRQMM_IM2COL_SMEM_KB=$1 LRQMM_IM2COL_MIN_TW=$2 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:im2col --csv --log-file gpurun_out/r6zm_${L}_$1_$2.csv python tools/one_layer.py $L 2 > /dev/null 2>&1
  echo "$L smem=$1 min_tw=$2: $(grep -h 'Kernel Name\|gpu__time' gpurun_out/r6zm_${L}_$1_$2.csv | grep -o 'im2col[a-z_]*\|"[0-9.]*"$' | tr '\n' ' ')" >> gpurun_out/r6zm.log
 done
done
LRQMM_IM2COL_SMEM_KB=100 LRQMM_IM2COL_MIN_TW=4 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k im2col > gpurun_out/r6zm_tests.log 2>&1; echo rc=$? >> gpurun_out/r6zm_tests.log
