# RSVD chain variants on c4 / c2 (separate launches vs cooperative apply vs fused passes)
for V in "" "LRQMM_RSVD_COOP=1" "LRQMM_RSVD_FUSED=1"; do
  tag=${V%%=*}; tag=${tag:-default}
  env $V timeout 900 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r4i_c4_$tag.json 2>&1
  env $V timeout 600 python bench.py --config c2 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r4i_c2_$tag.json 2>&1
done
