#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -rA -x -k "inverse or gauss" > gpurun_out/s2_pytest_gj.log 2>&1; echo "pytest gj rc=$?"; tail -3 gpurun_out/s2_pytest_gj.log
AIFMM_DEBUG_INV=1 python tools/gpu_perf.py 1 > gpurun_out/s2_inv_cfg2_fused.log 2>&1
AIFMM_DEBUG_INV=1 python tools/gpu_perf.py 2 > gpurun_out/s2_inv_cfg3_fused.log 2>&1
python tools/gpu_perf.py 2 2>&1 | tail -1 | cut -c1-400
python tools/gpu_perf.py 1 2>&1 | tail -1 | cut -c1-400
