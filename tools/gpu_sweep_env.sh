#!/bin/bash
# factor time of configs 2 and 3 under kernel-routing toggles
for env in "X=1" "AIFMM_HH_SMEM=1"; do
  for cfg in 1 2; do
    echo "$env cfg$cfg $(env $env timeout 600 python tools/gpu_perf.py $cfg 2>/dev/null | grep '^{' | tail -1 | cut -c1-150)"
  done
done
