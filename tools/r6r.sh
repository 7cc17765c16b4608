# Gram one-wave grid + apply64_tc per-block column maxima: kernels of layer1.0.conv3 (ncu full) + tests + c4
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_apply_small|k_apply64_tc|k_fused_small|k_split_bf16|k_tc_proj|k8_gemm" -c 24 -o gpurun_out/r6r_tall python tools/one_layer.py layer1.0.conv3 1 > gpurun_out/r6r.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r6r_tests.log 2>&1; echo rc=$? >> gpurun_out/r6r_tests.log
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r6r_bench_c4.json 2>&1
