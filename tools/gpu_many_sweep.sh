#!/bin/bash
# factor time of config 2 vs the one-CTA-per-task threshold (AIFMM_MANY)
for m in 296 96 32; do
  echo "AIFMM_MANY=$m"; AIFMM_MANY=$m timeout 300 python tools/gpu_perf.py 1 2>/dev/null | grep '^{' | tail -1 | cut -c1-160
done
