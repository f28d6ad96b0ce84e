#!/bin/bash
set -x
python -m pytest tests -m gpu -q -rA > gpurun_out/r02_pytest_gpu16.log 2>&1; echo "pytest rc=$?"
grep -E "config 3:|N=|GMRES iter|passed|failed|FAILED" gpurun_out/r02_pytest_gpu16.log | tail -10
python bench.py --cfg 3 --steps 3 --warmup 3 > gpurun_out/r02_bench_cfg3_g.log 2>&1; echo "bench3 rc=$?"
tail -1 gpurun_out/r02_bench_cfg3_g.log | cut -c1-400
python bench.py --cfg 2 --steps 5 --warmup 3 > gpurun_out/r02_bench_cfg2_g.log 2>&1; echo "bench2 rc=$?"
tail -1 gpurun_out/r02_bench_cfg2_g.log | cut -c1-300
bash tools/gpu_sanitize.sh
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg3_final2.csv \
  python bench.py --cfg 3 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r02_ncu_final2.log 2>&1; echo "ncu final rc=$?"
