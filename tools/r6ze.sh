# eigensolver n = 24 with 22 live columns: group sizes
./tools/eig_bench 2>&1 | grep "n=24" > gpurun_out/r6ze_eig.log
