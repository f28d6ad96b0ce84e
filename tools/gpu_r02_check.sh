#!/bin/bash
# round-2 GPU check: GPU tests, config-3 and config-2 bench lines, config-3 launch list
set -x
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv
free -g | head -2; nproc
python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02_pytest_gpu.log
python bench.py --cfg 3 --steps 3 --warmup 3 > gpurun_out/r02_bench_cfg3.log 2>&1; echo "bench3 rc=$?"
tail -2 gpurun_out/r02_bench_cfg3.log
python bench.py --cfg 2 --steps 5 --warmup 3 > gpurun_out/r02_bench_cfg2.log 2>&1; echo "bench2 rc=$?"
tail -1 gpurun_out/r02_bench_cfg2.log | cut -c1-400
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg3.csv \
  python bench.py --cfg 3 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r02_ncu_cfg3.log 2>&1; echo "ncu rc=$?"
