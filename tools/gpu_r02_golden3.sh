#!/bin/bash
# config-3 oracle golden on the GPU box's host (196 GB RAM, 16 cores), then the GPU tests
set -x
nproc; free -g | head -2; lscpu | grep "Model name"
python -c "from oracle.cpp import build; print(build(force=True))"
python tools/oracle_golden.py 3 16 0 gpurun_out > gpurun_out/r02_golden3.log 2>&1; echo "golden rc=$?"
tail -25 gpurun_out/r02_golden3.log
mkdir -p tests/golden && cp gpurun_out/cfg3_rand2d_matern_1M_oracle.npz tests/golden/ 2>/dev/null
python -m pytest tests -m gpu -q -rA -k "config3 or residual or algorithm2 or three_preconditioners" > gpurun_out/r02_pytest_gpu2.log 2>&1; echo "pytest rc=$?"
grep -E "config 3:|passed|failed|Error" gpurun_out/r02_pytest_gpu2.log | tail -15
