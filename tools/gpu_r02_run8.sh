#!/bin/bash
set -x
python -m pytest tests -m gpu -q -rA > gpurun_out/r02_pytest_gpu8.log 2>&1; echo "pytest rc=$?"
grep -E "config 3:|GMRES iter|passed|failed|FAILED" gpurun_out/r02_pytest_gpu8.log | tail -8
for env in "X=1" "AIFMM_NULLSPACE=1"; do
  for cfg in 2 1; do
    echo "$env cfg$cfg $(env $env timeout 600 python tools/gpu_perf.py $cfg 2>/dev/null | grep '^{' | tail -1)"
  done
done > gpurun_out/r02_ab8.log 2>&1
cut -c1-600 gpurun_out/r02_ab8.log
python tools/gpu_alg2.py 1 > gpurun_out/r02_alg2_cfg2.log 2>&1; cat gpurun_out/r02_alg2_cfg2.log
python tools/gpu_alg2.py 2 > gpurun_out/r02_alg2_cfg3.log 2>&1; cat gpurun_out/r02_alg2_cfg3.log
for n in 65536 131072 262144; do timeout 1500 python tools/gpu_cfg5_table.py $n 300 >> gpurun_out/r02_cfg5_table.log 2>&1; done
cat gpurun_out/r02_cfg5_table.log | cut -c1-900
timeout 1500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "schur/" --launch-skip 4 -c 8 -o /tmp/prof_schur -f \
    python tools/gpu_once.py 2 > gpurun_out/r02_ncu_schur.log 2>&1; echo "ncu schur rc=$?"
python tools/ncu_kernel_traffic.py /tmp/prof_schur.ncu-rep gpurun_out/r02_ncu_schur.json "gemm_tasks_kernel" | head -16
