# eigensolver live-size dispatch at n = 24 too: tests + c2/c3/c4
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r6zf_tests.log 2>&1; echo rc=$? >> gpurun_out/r6zf_tests.log
for c in c2 c3; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r6zf_bench_$c.json 2>&1; done
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r6zf_bench_c4.json 2>&1
