# stability: the GPU suite three times on the final build
for i in 1 2 3; do timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r6zi_tests_$i.log 2>&1; echo rc=$? >> gpurun_out/r6zi_tests_$i.log; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r6zi_smoke.log 2>&1; echo rc=$? >> gpurun_out/r6zi_smoke.log
