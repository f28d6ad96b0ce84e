#!/bin/bash
# factor time of configs 3 and 2 under TSQR chunking variants of the RRQR first stage
for env in "X=1" "AIFMM_TSQR_MMAX=100000 AIFMM_TSQR_ROWS=4096 AIFMM_TSQR_NMIN=4096" \
           "AIFMM_TSQR_MMAX=100000 AIFMM_TSQR_ROWS=4096 AIFMM_TSQR_NMIN=1024" \
           "AIFMM_TSQR_MMAX=100000 AIFMM_TSQR_ROWS=2048 AIFMM_TSQR_NMIN=2048" \
           "AIFMM_TSQR_MMAX=100000 AIFMM_TSQR_ROWS=1024 AIFMM_TSQR_NMIN=1024"; do
  for cfg in 2 1; do
    echo "$env cfg$cfg $(env $env timeout 600 python tools/gpu_perf.py $cfg 2>/dev/null | grep '^{' | tail -1)"
  done
done
