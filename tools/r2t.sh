timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2t_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2t_gpu.log
for L in layer1.0.conv3 conv1 layer1.0.conv2; do
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2t_launches_$L.csv python tools/one_layer.py $L 2 > /dev/null 2>&1
done
timeout 300 python bench.py --config c2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2t_bench_c2.json 2>&1
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 > gpurun_out/r2t_bench_c4.json 2>&1
