#!/bin/bash
# K7 raster-group / L2-policy sweep at c3: per setting the step phases (CUDA events) and the GEMM's
# DRAM bytes (ncu, one launch).  Settings: "GROUP POLA POLB".
for s in "8 2 0" "8 2 1" "8 2 0" "8 2 1" "6 2 1" "12 2 1" "8 0 1" "8 2 3" "10 2 1"; do
  set -- $s
  export LRQMM_G7_GROUP=$1 LRQMM_G7_POLA=$2 LRQMM_G7_POLB=$3
  t=$(python tools/time_phases.py --config c3 --steps 5 2>&1 | tail -1)
  d=$(ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k7_gemm -c 1 python tools/time_phases.py --config c3 --steps 1 2>&1 | grep -E "dram__bytes_read|hit_rate" | awk '{print $1"="$3$2}' | tr '\n' ' ')
  echo "group=$1 polA=$2 polB=$3: $t  $d"
done
