# k_fused_small phase stamps (trace build) at c2 and c3 and c4-like
for c in c2 c3; do LRQMM_LIB=tools/bin/liblrqmm_fstrace.so timeout 300 python tools/fs_trace.py --config $c >> gpurun_out/r6z_trace.log 2>&1; done
