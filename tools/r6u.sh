# fresh c4 launch list (after the assembly / solver changes)
timeout 2000 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r6u_c4_all.csv python tools/c4_all.py > gpurun_out/r6u_c4.log 2>&1
