# CholQR variants: pipelined Schur update (p) x select tree (t)
for b in tools/bin/eb_c_p*; do echo "== $b" >> gpurun_out/r6n_chol.log; $b 2>&1 | grep chol >> gpurun_out/r6n_chol.log; done
