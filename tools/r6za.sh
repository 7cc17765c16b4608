# Jacobi stopping threshold: steps, time, projector error vs numpy on the two fixtures
for t in 1e-16 1e-14 1e-12 1e-10; do
  echo "== tol $t" >> gpurun_out/r6za_tol.log
  ./tools/bin/eb_tol_$t 2>&1 | grep "NT=128\|NT=192\|NT=256" >> gpurun_out/r6za_tol.log
  python tools/eig_check.py tools/eig_G24.bin 24 16 gpurun_out/eig_T_256_n24.bin >> gpurun_out/r6za_tol.log 2>&1
  python tools/eig_check.py tools/eig_G32.bin 32 16 gpurun_out/eig_T_256_n32.bin >> gpurun_out/r6za_tol.log 2>&1
done
