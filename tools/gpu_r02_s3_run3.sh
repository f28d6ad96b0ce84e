#!/bin/bash
# split trailing-update pipeline variants (shared memory -> CTAs per SM): bitwise + timing
for c in 2 1; do
  for v in "3 3" "2 3" "4 3" "3 2" "2 2" "4 2"; do
    set -- $v
    AIFMM_HHU_P1=$1 AIFMM_HHU_P2=$2 python tools/gpu_xhash.py $c 2 | tail -1 | sed "s/^/p1=$1 p2=$2 /"
  done
done
