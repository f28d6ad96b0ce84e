#!/bin/bash
# distributed factorization, in-process multi-rank emulation on one GPU
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -rA -x -s > gpurun_out/s2_pytest_dist.log 2>&1; echo "pytest dist rc=$?"
grep -E "world|passed|failed|FAILED|Error|error" gpurun_out/s2_pytest_dist.log | tail -20
