# binding getters ordered against the handle stream + image dedup: the failing sequence, then the full suite x3
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_multirank.py -q > gpurun_out/r5m_seq.log 2>&1; echo rc=$? >> gpurun_out/r5m_seq.log
for i in 1 2 3; do
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r5m_full_$i.log 2>&1; echo rc=$? >> gpurun_out/r5m_full_$i.log
done
