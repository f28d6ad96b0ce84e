#!/bin/bash
# config-5 preconditioner quality vs N (symmetric reading R27 vs independent sides)
for n in 65536 131072 262144; do
  echo "sym n=$n $(timeout 900 python tools/gpu_cfg5_diag.py $n 128 2>&1 | grep '^{' | tail -1)"
done
echo "asym n=131072 $(AIFMM_ASYMMETRIC=1 timeout 900 python tools/gpu_cfg5_diag.py 131072 128 2>&1 | grep '^{' | tail -1)"
