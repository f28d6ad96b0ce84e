#!/bin/bash
# config-3 golden with the R8c oracle (box host), then the GPU suite and the A/B of the defaults
set -x
python -c "from oracle.cpp import build; print(build(force=True))"
python tools/oracle_golden.py 3 16 0 gpurun_out > gpurun_out/r02_golden3b.log 2>&1; echo "golden rc=$?"
tail -1 gpurun_out/r02_golden3b.log | cut -c1-400
cp gpurun_out/cfg3_rand2d_matern_1M_oracle.npz tests/golden/
python -m pytest tests -m gpu -q -rA > gpurun_out/r02_pytest_gpu13.log 2>&1; echo "pytest rc=$?"
grep -E "config 3:|N=|GMRES iter|passed|failed|FAILED" gpurun_out/r02_pytest_gpu13.log | tail -10
for env in "X=1" "AIFMM_NULLSPACE=0" "AIFMM_SYM_SCHUR=1"; do
  for cfg in 2 1; do
    echo "$env cfg$cfg $(env $env timeout 600 python tools/gpu_perf.py $cfg 2>/dev/null | grep '^{' | tail -1)"
  done
done > gpurun_out/r02_ab13.log 2>&1
cut -c1-700 gpurun_out/r02_ab13.log
