#!/bin/bash
set -x
python -m pytest tests -m gpu -q -rA > gpurun_out/r02_pytest_gpu14.log 2>&1; echo "pytest rc=$?"
grep -E "config 3:|N=|GMRES iter|passed|failed|FAILED" gpurun_out/r02_pytest_gpu14.log | tail -10
python bench.py --cfg 3 --steps 3 --warmup 3 > gpurun_out/r02_bench_cfg3_f.log 2>&1; echo "bench3 rc=$?"
tail -1 gpurun_out/r02_bench_cfg3_f.log | cut -c1-700
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
