#!/bin/bash
# ncu durations (boost clocks) of the fused small-solver kernel: W in {24,32}, op 3 (CholQR) / 4 (eig)
for W in 24 32; do for op in 3 4; do
  python tools/prof_small.py $W $op 2048 > /dev/null
  t=$(ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_fused_small python tools/prof_small.py $W $op 2048 1 2>&1 | grep duration | awk '{print $3}')
  echo "W=$W op=$op fused_small: $t us"
done; done
