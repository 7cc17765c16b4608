# GEMM kernel choice at c2 / c4: auto vs K6 vs K7 vs K8
for V in 0 1 2 3; do
LRQMM_GEMM_VARIANT=$V timeout 300 python bench.py --config c2 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r3y_c2_v$V.json 2>&1
done
for V in 0 2; do
LRQMM_GEMM_VARIANT=$V timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r3y_c4_v$V.json 2>&1
done
