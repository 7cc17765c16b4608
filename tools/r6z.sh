# k_fused_small phase stamps + Jacobi step count (trace build) at c2 / c3 and one c4 layer
for c in c2 c3; do LRQMM_LIB=tools/bin/liblrqmm_fstrace.so timeout 300 python tools/fs_trace.py --config $c >> gpurun_out/r6z_trace.log 2>&1; done
