#!/bin/bash
# workspace budget 48 GB default: GPU suite + smoke + config-3 bench
python -m pytest tests -m gpu -q -rA > gpurun_out/s2_pytest_gpu9.log 2>&1; echo "pytest rc=$?"
grep -E "config 2:|config 3:|passed|failed|FAILED|XPASS" gpurun_out/s2_pytest_gpu9.log | tail -8
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 3 --warmup 3 > gpurun_out/s2_bench_cfg3.log 2>&1; echo "bench3 rc=$?"; tail -1 gpurun_out/s2_bench_cfg3.log | cut -c1-700
