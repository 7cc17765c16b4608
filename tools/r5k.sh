# multirank flake check: new build x3, previous build x3
for i in 1 2 3; do
timeout 600 python -m pytest tests/test_gpu_multirank.py -q > gpurun_out/r5k_new_$i.log 2>&1; echo rc=$? >> gpurun_out/r5k_new_$i.log
LRQMM_LIB=$PWD/paper_2409_18772_b200/liblrqmm_prev.so timeout 600 python -m pytest tests/test_gpu_multirank.py -q > gpurun_out/r5k_prev_$i.log 2>&1; echo rc=$? >> gpurun_out/r5k_prev_$i.log
done
