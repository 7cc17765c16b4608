# one ncu --set full capture of the c3 GEMM (K7) with the final build (roofline traffic)
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k7_gemm --launch-skip 1 -c 1 -o gpurun_out/r6zp_gemm_c3 python tools/one_step.py --config c3 --steps 2 > gpurun_out/r6zp.log 2>&1
