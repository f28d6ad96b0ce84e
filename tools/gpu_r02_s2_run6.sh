#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -rA -x > gpurun_out/s2_pytest_kern.log 2>&1; echo "pytest kernels rc=$?"; tail -2 gpurun_out/s2_pytest_kern.log
AIFMM_DEBUG_INV=1 python tools/gpu_perf.py 1 > gpurun_out/s2_inv_cfg2_v2.log 2>&1
AIFMM_DEBUG_INV=1 python tools/gpu_perf.py 2 > gpurun_out/s2_inv_cfg3_v2.log 2>&1
AIFMM_DEBUG_INV=1 AIFMM_GJ_FUSED_MIN=0 python tools/gpu_perf.py 2 > gpurun_out/s2_inv_cfg3_v2_nofused.log 2>&1
python tools/gpu_perf.py 2 2>&1 | tail -1 | cut -c1-300
AIFMM_GJ_FUSED_MIN=0 python tools/gpu_perf.py 2 2>&1 | tail -1 | cut -c1-300
python tools/gpu_perf.py 1 2>&1 | tail -1 | cut -c1-300
