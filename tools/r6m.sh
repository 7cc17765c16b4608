# CholQR v2 (pipelined Schur update, select tree, MUFU rsqrt + Newton, branch-free transform): phase clocks + timing
./tools/bin/eb_cprof2 2>&1 | grep chol > gpurun_out/r6m_chol.log
./tools/bin/eb_chol2 2>&1 | grep chol >> gpurun_out/r6m_chol.log
