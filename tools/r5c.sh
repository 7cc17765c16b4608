# K1 TMA with two consumer groups for K = 4096 rows: parity, c2 bench A/B
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "quantize or lrqmm_matches" > gpurun_out/r5c_tests.log 2>&1; echo rc=$? >> gpurun_out/r5c_tests.log
for G in 2 1; do
LRQMM_K1_GROUPS=$G timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k1_quantize --csv --log-file gpurun_out/r5c_k1_g$G.csv python tools/one_step.py --config c2 --steps 2 > /dev/null 2>&1
LRQMM_K1_GROUPS=$G timeout 600 python bench.py --config c2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r5c_bench_c2_g$G.json 2>&1
done
