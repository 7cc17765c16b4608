for L in layer1.0.conv3 layer1.0.conv2 conv1 layer3.0.conv2; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2m_launches_$L.csv python tools/one_layer.py $L 2 > gpurun_out/r2m_$L.log 2>&1
done
