#!/bin/bash
# look-ahead trailing-update schedule (second stream) vs default: bitwise + timing
for c in 2 1 0; do
  python tools/gpu_xhash.py $c 2 | tail -1 | sed "s/^/default   /"
  AIFMM_HHU_LOOKAHEAD=1 python tools/gpu_xhash.py $c 3 | tail -2 | sed "s/^/lookahead /"
done
