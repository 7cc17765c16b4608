# fused Gram finisher: partial sums with batched loads
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r6v_tests.log 2>&1; echo rc=$? >> gpurun_out/r6v_tests.log
for c in c2 c3; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r6v_bench_$c.json 2>&1; done
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r6v_bench_c4.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r6v_l4.csv python tools/one_layer.py layer4.2.conv3 2 > /dev/null 2>&1
