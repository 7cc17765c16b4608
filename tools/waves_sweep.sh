#!/bin/bash
# RSVD pass work units per SM (split-K factor) sweep at a config: tools/waves_sweep.sh [config]
for w in 6 1 2 3 4 6 8; do
  echo "waves=$w: $(LRQMM_TC_WAVES=$w python tools/time_phases.py --config ${1:-c3} --steps 10 2>&1 | tail -1)"
done
