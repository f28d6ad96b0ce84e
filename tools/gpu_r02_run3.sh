#!/bin/bash
# GPU tests with the symmetric Schur updates, TSQR sweep, bench line, then the config-3 oracle golden
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu3.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02_pytest_gpu3.log
bash tools/gpu_sweep_tsqr.sh > gpurun_out/r02_sweep_tsqr.log 2>&1
cat gpurun_out/r02_sweep_tsqr.log | cut -c1-330
python bench.py --cfg 3 --steps 3 --warmup 3 > gpurun_out/r02_bench_cfg3_b.log 2>&1; echo "bench3 rc=$?"
tail -1 gpurun_out/r02_bench_cfg3_b.log | cut -c1-700
python -c "from oracle.cpp import build; print(build(force=True))"
python tools/oracle_golden.py 3 16 0 gpurun_out > gpurun_out/r02_golden3.log 2>&1; echo "golden rc=$?"
tail -5 gpurun_out/r02_golden3.log | cut -c1-600
mkdir -p tests/golden && cp gpurun_out/cfg3_rand2d_matern_1M_oracle.npz tests/golden/ 2>/dev/null
python -m pytest tests -m gpu -q -rA -k "config3" > gpurun_out/r02_pytest_cfg3.log 2>&1; echo "pytest cfg3 rc=$?"
grep -E "config 3:|passed|failed|Error" gpurun_out/r02_pytest_cfg3.log | tail -8
