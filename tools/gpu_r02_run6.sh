#!/bin/bash
# GPU suite; A/B of R30 (symmetric Schur) and R31 (null-space pivots, opt-in); TSQR sweep
set -x
python -m pytest tests -m gpu -q -rA -x > gpurun_out/r02_pytest_gpu6.log 2>&1; echo "pytest rc=$?"
grep -E "config 3:|GMRES iter|passed|failed|FAILED" gpurun_out/r02_pytest_gpu6.log | tail -8
for env in "X=1" "AIFMM_NO_SYM_SCHUR=1" "AIFMM_NULLSPACE=1" "X=2" "AIFMM_NO_SYM_SCHUR=2"; do
  for cfg in 2 1; do
    echo "$env cfg$cfg $(env $env timeout 600 python tools/gpu_perf.py $cfg 2>/dev/null | grep '^{' | tail -1)"
  done
done > gpurun_out/r02_ab6.log 2>&1
cut -c1-420 gpurun_out/r02_ab6.log
bash tools/gpu_sweep_tsqr.sh > gpurun_out/r02_sweep_tsqr6.log 2>&1
cut -c1-420 gpurun_out/r02_sweep_tsqr6.log
