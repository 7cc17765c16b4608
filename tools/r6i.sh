# eigensolver: step loop unrolled by two (static ping-pong addresses)
./tools/bin/eb_unroll > gpurun_out/r6i_eig.log 2>&1
python tools/eig_check.py tools/eig_G24.bin 24 16 gpurun_out/eig_T_256_n24.bin >> gpurun_out/r6i_eig.log 2>&1
python tools/eig_check.py tools/eig_G32.bin 32 16 gpurun_out/eig_T_256_n32.bin >> gpurun_out/r6i_eig.log 2>&1
