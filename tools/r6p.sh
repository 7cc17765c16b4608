# c4 / c2 with the opt-in fused passes and the cooperative apply (after the solver speedups)
for v in FUSED COOP; do
  env LRQMM_RSVD_$v=1 timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r6p_c4_$v.json 2>&1
  env LRQMM_RSVD_$v=1 timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r6p_c2_$v.json 2>&1
done
