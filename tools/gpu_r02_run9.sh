#!/bin/bash
set -x
for env in "X=1" "AIFMM_PQR_MANY_MMAX=700" "AIFMM_PQR_MANY_MMAX=1200" "AIFMM_HHU_ST=64" "AIFMM_HHU_ST=2"; do
  for cfg in 2 1; do
    echo "$env cfg$cfg $(env $env timeout 600 python tools/gpu_perf.py $cfg 2>/dev/null | grep '^{' | tail -1)"
  done
done > gpurun_out/r02_ab9.log 2>&1
cut -c1-640 gpurun_out/r02_ab9.log
timeout 1500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "schur/" --launch-skip 4 -c 6 -o /tmp/prof_schur -f \
    python tools/gpu_once.py 2 > gpurun_out/r02_ncu_schur.log 2>&1; echo "ncu schur rc=$?"
python tools/ncu_kernel_traffic.py /tmp/prof_schur.ncu-rep gpurun_out/r02_ncu_schur.json "gemm_tasks_kernel" | head -24
ls -la /tmp/prof_schur.ncu-rep
