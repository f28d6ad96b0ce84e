#!/bin/bash
# Gauss-Jordan routing sweep on config 3 / 2: cluster panels for larger batches
for v in "148 0" "300 0" "300 2" "1100 2" "1100 4"; do set -- $v
  echo "cluster_max=$1 cl=$2"
  AIFMM_GJ_CLUSTER_MAX=$1 AIFMM_GJ_CL=$2 AIFMM_DEBUG_INV=1 python tools/gpu_perf.py 2 > gpurun_out/s2_gjsweep_$1_$2.log 2>&1
  tail -1 gpurun_out/s2_gjsweep_$1_$2.log | cut -c1-200
done
