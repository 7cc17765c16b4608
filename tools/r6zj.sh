# K8 epilogue anatomy on layer1.0.conv3 (N = 256, K = 64): no D stores (1), no TMEM loads (2), neither (3)
for v in 0 1 2 3; do
  lib=paper_2409_18772_b200/liblrqmm.so; [ $v != 0 ] && lib=tools/bin/liblrqmm_k8exp$v.so
  LRQMM_LIB=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k8_gemm --csv --log-file gpurun_out/r6zj_$v.csv python tools/one_layer.py layer1.0.conv3 2 > /dev/null 2>&1
  echo "exp $v: $(grep -h gpu__time_duration gpurun_out/r6zj_$v.csv | awk -F'","' '{gsub(/"/,"",$NF); printf "%.1f ", $NF/1000}')" >> gpurun_out/r6zj.log
done
