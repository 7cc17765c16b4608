# eigensolver: group-uniform skip of dead block / V slots (n = 32 at NT = 192)
./tools/bin/eb_skipu > gpurun_out/r6j_eig.log 2>&1
python tools/eig_check.py tools/eig_G24.bin 24 16 gpurun_out/eig_T_256_n24.bin >> gpurun_out/r6j_eig.log 2>&1
python tools/eig_check.py tools/eig_G32.bin 32 16 gpurun_out/eig_T_256_n32.bin >> gpurun_out/r6j_eig.log 2>&1
