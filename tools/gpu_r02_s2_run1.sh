#!/bin/bash
# session-2 baseline: GPU suite, smoke, config-3 and config-2 bench lines at HEAD
python -m pytest tests -m gpu -q -rA -x > gpurun_out/s2_pytest_gpu1.log 2>&1; echo "pytest rc=$?"
grep -E "config 2:|config 3:|passed|failed|FAILED" gpurun_out/s2_pytest_gpu1.log | tail -10
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 3 --warmup 3 > gpurun_out/s2_bench_cfg3.log 2>&1; echo "bench3 rc=$?"; tail -1 gpurun_out/s2_bench_cfg3.log | cut -c1-600
python bench.py --cfg 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s2_bench_cfg2.log 2>&1; echo "bench2 rc=$?"; tail -1 gpurun_out/s2_bench_cfg2.log | cut -c1-600
