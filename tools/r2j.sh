timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2j_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2j_gpu.log
timeout 600 python tools/cublaslt_int8.py gpurun_out/r02_cublaslt_int8.json > gpurun_out/r2j_lt.log 2>&1
timeout 900 python tools/paper_sweeps.py rank qt tables --out gpurun_out/r02 > gpurun_out/r2j_sweeps.log 2>&1
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/one_step.py --config c1 --steps 2 > gpurun_out/r02_sanitizer_memcheck_c1.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/one_step.py --config c2 --steps 1 > gpurun_out/r02_sanitizer_memcheck_c2.log 2>&1
timeout 600 compute-sanitizer --tool synccheck --print-limit 20 python tools/one_step.py --config c1 --steps 2 > gpurun_out/r02_sanitizer_synccheck_c1.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "lrqmm_matches_oracle and normal and 4-" > gpurun_out/r02_sanitizer_memcheck_parity.log 2>&1
