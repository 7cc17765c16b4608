# G' reduction deferred to the cross-Gram branch: tests, A/B at c2 and c3, c4 bench
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x > gpurun_out/r5o_tests.log 2>&1; echo rc=$? >> gpurun_out/r5o_tests.log
bash tools/ab.sh $PWD/paper_2409_18772_b200/liblrqmm_prev.so $PWD/paper_2409_18772_b200/liblrqmm.so c2 3 > gpurun_out/r5o_ab_c2.log 2>&1
bash tools/ab.sh $PWD/paper_2409_18772_b200/liblrqmm_prev.so $PWD/paper_2409_18772_b200/liblrqmm.so c3 2 > gpurun_out/r5o_ab_c3.log 2>&1
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r5o_bench_c4.json 2>&1
