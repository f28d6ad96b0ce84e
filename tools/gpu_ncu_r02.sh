#!/bin/bash
# ncu --set full captures (config 3, one build+factor+solve) of the dominant kernels, summarised
# by tools/ncu_kernel_traffic.py into gpurun_out/r02_ncu_*.json (copied to profiles/ afterwards)
set -x
cap() {  # name, ncu filter args..., kernel regex for the summary
  local name=$1; shift; local rx=$1; shift
  timeout 1500 ncu --set full --clock-control none --import-source on "$@" -o /tmp/prof_$name -f \
    python tools/gpu_once.py 2 > gpurun_out/r02_ncu_$name.log 2>&1; echo "ncu $name rc=$?"
  python tools/ncu_kernel_traffic.py /tmp/prof_$name.ncu-rep gpurun_out/r02_ncu_$name.json "$rx" > /dev/null 2>&1
  cat gpurun_out/r02_ncu_$name.json | head -14
}
cap schur "gemm_tasks_kernel" --nvtx --nvtx-include "schur/" --launch-skip 4 -c 8
cap hhupdate "hh_update" -k regex:hh_update --launch-skip 400 -c 8
cap hhpanel "hh_panel" -k regex:hh_panel_cluster_kernel --launch-skip 100 -c 6
cap pqr "pqr" -k regex:pqr_cluster --launch-skip 10 -c 4
cap gj "gj_" -k regex:gj_panel --launch-skip 50 -c 8
cap aca "aca_kernel" -k regex:aca_kernel --launch-skip 2 -c 2
