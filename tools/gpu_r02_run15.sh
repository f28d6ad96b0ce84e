#!/bin/bash
set -x
for env in "X=1" "AIFMM_NULLSPACE=2 AIFMM_NULLSPACE_PMAX=16" "AIFMM_NULLSPACE=2 AIFMM_NULLSPACE_PMAX=32" "AIFMM_NULLSPACE=2 AIFMM_NULLSPACE_PMAX=64" "AIFMM_NULLSPACE=2 AIFMM_NULLSPACE_PMAX=128"; do
  for cfg in 2 1; do
    echo "$env cfg$cfg $(env $env timeout 600 python tools/gpu_perf.py $cfg 2>/dev/null | grep '^{' | tail -1)"
  done
done > gpurun_out/r02_ab15.log 2>&1
cut -c1-720 gpurun_out/r02_ab15.log
