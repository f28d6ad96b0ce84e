#!/bin/bash
set -x
python tools/gpu_perf.py 2 | tail -1
python tools/gpu_perf.py 1 | tail -1
python bench.py --cfg 3 --steps 3 --warmup 3 > gpurun_out/r02_bench_cfg3_h.log 2>&1; echo "bench3 rc=$?"
tail -1 gpurun_out/r02_bench_cfg3_h.log | cut -c1-300
