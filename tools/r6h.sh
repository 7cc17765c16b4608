# eigensolver: thread-group sizes and step anatomy (skip variants at 4 fixed sweeps)
./tools/bin/eb_s0_w0 > gpurun_out/r6h_eig.log 2>&1
python tools/eig_check.py tools/eig_G24.bin 24 16 gpurun_out/eig_T_256_n24.bin >> gpurun_out/r6h_eig.log 2>&1
python tools/eig_check.py tools/eig_G32.bin 32 16 gpurun_out/eig_T_256_n32.bin >> gpurun_out/r6h_eig.log 2>&1
for b in tools/bin/eb_s*_w4; do echo "== $b" >> gpurun_out/r6h_skip.log; $b 2>&1 | grep "NT=256\|NT=128" >> gpurun_out/r6h_skip.log; done
