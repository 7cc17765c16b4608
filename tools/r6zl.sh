# c4 launch list of the final build (per-kernel totals)
timeout 2000 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r6zl_c4_all.csv python tools/c4_all.py > gpurun_out/r6zl_c4.log 2>&1
