# eigensolver step anatomy: new step (branch-free, split V update) and skip variants at 4 fixed sweeps
./tools/eig_bench > gpurun_out/r6g_eig_new.log 2>&1
python tools/eig_check.py tools/eig_G24.bin 24 16 gpurun_out/eig_T_256_n24.bin >> gpurun_out/r6g_eig_new.log 2>&1
python tools/eig_check.py tools/eig_G32.bin 32 16 gpurun_out/eig_T_256_n32.bin >> gpurun_out/r6g_eig_new.log 2>&1
for b in gpurun_out/eb_s*; do echo "== $b" >> gpurun_out/r6g_skip.log; $b 2>&1 | grep "NT=256" >> gpurun_out/r6g_skip.log; done
