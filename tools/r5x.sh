# staggered range-finder branches: tests with the stagger on, A/B timing
LRQMM_BRANCH_STAGGER=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -q -x > gpurun_out/r5x_tests.log 2>&1; echo rc=$? >> gpurun_out/r5x_tests.log
for i in 1 2; do for S in 0 1; do
  LRQMM_BRANCH_STAGGER=$S timeout 600 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r5x_c3_s${S}_$i.json 2>&1
  LRQMM_BRANCH_STAGGER=$S timeout 600 python bench.py --config c2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r5x_c2_s${S}_$i.json 2>&1
done; done
for S in 0 1; do LRQMM_BRANCH_STAGGER=$S timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r5x_c4_s$S.json 2>&1; done
