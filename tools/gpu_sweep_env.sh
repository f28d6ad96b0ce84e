#!/bin/bash
# factor time of configs 2 and 3 under a kernel-variant toggle
for env in "X=1" "AIFMM_GEMM_WIDE=1" "X=2" "AIFMM_GEMM_WIDE=2"; do
  for cfg in 1 2; do
    echo "$env cfg$cfg $(env $env timeout 600 python tools/gpu_perf.py $cfg 2>/dev/null | grep '^{' | tail -1 | cut -c1-150)"
  done
done
