#!/bin/bash
# factor time + residual of config 2 under debug toggles of the compression stage
for env in "X=1" "AIFMM_NO_TSQR=1" "AIFMM_TSQR_MMAX=64" "AIFMM_TSQR_MMAX=100000" "AIFMM_HH_CLUSTER=1"; do
  echo "$env $(env $env timeout 600 python tools/gpu_perf.py 1 2>/dev/null | grep -E '^\{|residual' | tail -2 | cut -c1-110 | tr '\n' ' ')"
done
