#!/bin/bash
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -rA -x -s > gpurun_out/s2_pytest_dist.log 2>&1; echo "pytest dist rc=$?"
grep -E "world|passed|failed|FAILED|Error|error" gpurun_out/s2_pytest_dist.log | tail -12
python bench.py --cfg 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s2_bench_cfg2.log 2>&1; echo "bench2 rc=$?"; tail -1 gpurun_out/s2_bench_cfg2.log | cut -c1-300
