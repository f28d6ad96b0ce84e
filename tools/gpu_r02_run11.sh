#!/bin/bash
set -x
python -m pytest tests -m gpu -q -rA -k "reduced_config or opt_in" > gpurun_out/r02_pytest_gpu11.log 2>&1; echo "pytest rc=$?"
grep -E "N=|passed|failed|FAILED|SKIPPED" gpurun_out/r02_pytest_gpu11.log | tail -8
AIFMM_NULLSPACE=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg3_r31.csv \
  python tools/gpu_once.py 2 > gpurun_out/r02_ncu_r31.log 2>&1; echo "ncu r31 rc=$?"
python tools/ncu_summary.py gpurun_out/r02_launches_cfg3_r31.csv | head -30
python bench.py --cfg 3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg3_final.csv \
  python bench.py --cfg 3 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r02_ncu_final.log 2>&1; echo "ncu final rc=$?"
python tools/ncu_summary.py gpurun_out/r02_launches_cfg3_final.csv | head -30
