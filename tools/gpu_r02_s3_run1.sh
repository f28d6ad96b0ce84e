#!/bin/bash
# hh_update split-pass variant: bitwise and timing against the fused kernel (config 3, config 2)
for c in 2 1; do
  AIFMM_HHU_SPLIT=0 python tools/gpu_xhash.py $c 2 | tail -1 | sed 's/^/fused     /'
  python tools/gpu_xhash.py $c 2 | tail -1 | sed 's/^/split296  /'
  AIFMM_HHU_SEG=512 python tools/gpu_xhash.py $c 2 | tail -1 | sed 's/^/seg512    /'
  AIFMM_HHU_SPLIT=100000 python tools/gpu_xhash.py $c 2 | tail -1 | sed 's/^/splitall  /'
done
