#!/bin/bash
# config-5 preconditioner quality vs N (current defaults)
for n in 65536 131072 262144; do
  echo "n=$n $(timeout 900 python tools/gpu_cfg5_diag.py $n 128 2>&1 | grep '^{' | tail -1)"
done
