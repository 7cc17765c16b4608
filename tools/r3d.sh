for R in 0 8 16 32; do
LRQMM_BRANCH_SMS=$R timeout 600 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r3d_c3_$R.json 2>&1
LRQMM_BRANCH_SMS=$R timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r3d_c2_$R.json 2>&1
done
