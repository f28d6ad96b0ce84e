#!/bin/bash
set -x
python -m pytest tests -m gpu -q -rA > gpurun_out/r02_pytest_gpu10.log 2>&1; echo "pytest rc=$?"
grep -E "config 3:|GMRES iter|passed|failed|FAILED" gpurun_out/r02_pytest_gpu10.log | tail -8
for env in "X=1" "AIFMM_FULL_RECORDS=1"; do
  for cfg in 2 1; do
    echo "$env cfg$cfg $(env $env timeout 600 python tools/gpu_perf.py $cfg 2>/dev/null | grep '^{' | tail -1)"
  done
done > gpurun_out/r02_ab10.log 2>&1
cut -c1-640 gpurun_out/r02_ab10.log
python bench.py --cfg 3 --steps 3 --warmup 3 > gpurun_out/r02_bench_cfg3_e.log 2>&1; echo "bench3 rc=$?"
tail -1 gpurun_out/r02_bench_cfg3_e.log | cut -c1-600
python bench.py --cfg 2 --steps 5 --warmup 3 > gpurun_out/r02_bench_cfg2_e.log 2>&1; echo "bench2 rc=$?"
tail -1 gpurun_out/r02_bench_cfg2_e.log | cut -c1-400
python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/r02_bench_ref.log 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/r02_bench_ref.log | cut -c1-500
