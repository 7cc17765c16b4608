# eigensolver: branch-free step, 3-MUFU rotation (A/B against the previous build) + MUFU latencies
./tools/lat > gpurun_out/r6f_lat.log 2>&1
./tools/eig_bench_old > gpurun_out/r6f_eig_old.log 2>&1
./tools/eig_bench > gpurun_out/r6f_eig_new.log 2>&1
python tools/eig_check.py tools/eig_G24.bin 24 16 gpurun_out/eig_T_256_n24.bin >> gpurun_out/r6f_eig_new.log 2>&1
python tools/eig_check.py tools/eig_G32.bin 32 16 gpurun_out/eig_T_256_n32.bin >> gpurun_out/r6f_eig_new.log 2>&1
