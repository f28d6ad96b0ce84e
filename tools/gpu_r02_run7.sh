#!/bin/bash
set -x
python -m pytest tests -m gpu -q -rA > gpurun_out/r02_pytest_gpu7.log 2>&1; echo "pytest rc=$?"
grep -E "config 3:|GMRES iter|passed|failed|FAILED" gpurun_out/r02_pytest_gpu7.log | tail -8
python tools/gpu_perf.py 2 | tail -1 | cut -c1-900
python tools/gpu_perf.py 1 | tail -1 | cut -c1-900
python bench.py --cfg 3 --steps 3 --warmup 3 > gpurun_out/r02_bench_cfg3_d.log 2>&1; echo "bench3 rc=$?"
tail -1 gpurun_out/r02_bench_cfg3_d.log
bash tools/gpu_ncu_r02.sh
