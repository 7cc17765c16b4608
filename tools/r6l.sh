# CholQR phase clocks
./tools/bin/eb_cprof 2>&1 | grep chol > gpurun_out/r6l_chol.log
