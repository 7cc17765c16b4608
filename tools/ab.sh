#!/bin/bash
# A/B of two liblrqmm builds in one session: tools/ab.sh A.so B.so [config] [rounds]
# (alternates, so clock / thermal drift hits both); prints the per-phase CUDA-event times.
A=$1; B=$2; CFG=${3:-c3}; R=${4:-3}
for i in $(seq $R); do
  for L in $A $B; do
    echo "$(basename $L): $(LRQMM_LIB=$L python tools/time_phases.py --config $CFG --steps 10 2>&1 | tail -1)"
  done
done
