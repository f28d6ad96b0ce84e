#!/bin/bash
set -x
python -m pytest tests -m gpu -q -rA -k "opt_in" > gpurun_out/r02_pytest_gpu12.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED" gpurun_out/r02_pytest_gpu12.log | tail -4
for env in "X=1" "AIFMM_NULLSPACE=1" "AIFMM_NULLSPACE=1 AIFMM_SYM_SCHUR=1"; do
  for cfg in 2 1; do
    echo "$env cfg$cfg $(env $env timeout 600 python tools/gpu_perf.py $cfg 2>/dev/null | grep '^{' | tail -1)"
  done
done > gpurun_out/r02_ab12.log 2>&1
cut -c1-700 gpurun_out/r02_ab12.log
