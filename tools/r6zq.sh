# c2 K1 consumer groups (4096-column rows)
for g in 1 2 4; do LRQMM_K1_GROUPS=$g timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r6zq_c2_g$g.json 2>&1; done
