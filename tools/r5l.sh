# full GPU suite x3 on the committed build (flake hunt)
for i in 1 2 3; do
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r5l_full_$i.log 2>&1; echo rc=$? >> gpurun_out/r5l_full_$i.log
done
