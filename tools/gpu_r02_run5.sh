#!/bin/bash
# full GPU suite (R30 fixed, R31), config-3 parity against the golden, bench lines
set -x
python -m pytest tests -m gpu -q -rA > gpurun_out/r02_pytest_gpu5.log 2>&1; echo "pytest rc=$?"
grep -E "config 3:|GMRES iter|passed|failed|FAILED" gpurun_out/r02_pytest_gpu5.log | tail -15
python tools/gpu_perf.py 2 > gpurun_out/r02_perf_cfg3.log 2>&1; tail -1 gpurun_out/r02_perf_cfg3.log
AIFMM_NO_SYM_SCHUR=1 python tools/gpu_perf.py 2 | tail -1
AIFMM_NO_NULLSPACE=1 python tools/gpu_perf.py 2 | tail -1
python tools/gpu_perf.py 1 | tail -1
AIFMM_NO_NULLSPACE=1 AIFMM_NO_SYM_SCHUR=1 python tools/gpu_perf.py 1 | tail -1
python bench.py --cfg 3 --steps 3 --warmup 3 > gpurun_out/r02_bench_cfg3_c.log 2>&1; echo "bench3 rc=$?"
tail -1 gpurun_out/r02_bench_cfg3_c.log | cut -c1-900
