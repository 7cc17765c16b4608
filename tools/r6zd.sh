# eigensolver n = 32 with 26 live columns on 192 threads: bench + projector check, tests, c4
./tools/eig_bench 2>&1 | grep "NT=" > gpurun_out/r6zd_eig.log
python tools/eig_check.py tools/eig_G32.bin 32 16 gpurun_out/eig_T_256_n32.bin >> gpurun_out/r6zd_eig.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r6zd_tests.log 2>&1; echo rc=$? >> gpurun_out/r6zd_tests.log
timeout 600 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r6zd_bench_c4.json 2>&1
