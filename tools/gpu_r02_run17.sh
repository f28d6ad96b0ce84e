#!/bin/bash
set -x
for env in "X=1" "AIFMM_ACA_SMEM_KB=40" "AIFMM_ACA_SMEM_KB=75" "AIFMM_ACA_SMEM_KB=110"; do
  for cfg in 2 1; do
    echo "$env cfg$cfg $(env $env timeout 600 python tools/gpu_perf.py $cfg 2>/dev/null | grep '^{' | tail -1 | cut -c1-160)"
  done
done
