# S1 pass (first k_tc_proj launch) and S3 dual pass on a tall layer: ncu full
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_tc_proj -s 0 -c 1 -o gpurun_out/r4f_s1 python tools/one_layer.py layer1.0.conv3 1 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_tc_proj -s 4 -c 1 -o gpurun_out/r4f_s3 python tools/one_layer.py layer1.0.conv3 1 > /dev/null 2>&1
