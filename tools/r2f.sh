ncu --set full --import-source on --clock-control none -k regex:k_tc_proj -c 1 -s 3 -o gpurun_out/r2f_s1_c2 python tools/one_step.py --config c2 --steps 2 > gpurun_out/r2f_ncu.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_apply_prep -c 1 -s 5 -o gpurun_out/r2f_ap_c2 python tools/one_step.py --config c2 --steps 2 >> gpurun_out/r2f_ncu.log 2>&1
