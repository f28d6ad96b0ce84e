#!/bin/bash
set -x
python -m pytest tests -m gpu -q -rA -k "reduced_config or deterministic" > gpurun_out/r02_pytest_gpu18.log 2>&1; echo "pytest rc=$?"
grep -E "N=|passed|failed|FAILED|Error" gpurun_out/r02_pytest_gpu18.log | tail -8
