# eigensolver micro-benchmark: steps / time at n = 24 (c2 sketch) and n = 32 (c4-like); ncu source view
./tools/eig_bench > gpurun_out/r3j_eig.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_bench -c 1 -o gpurun_out/r3j_eig256 ./tools/eig_bench > /dev/null 2>&1
