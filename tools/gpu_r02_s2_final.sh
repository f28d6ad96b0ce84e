#!/bin/bash
# session-2 final: GPU suite, smoke, config-3 / config-2 bench lines, reference arm
python -m pytest tests -m gpu -q -rA > gpurun_out/s2_pytest_final.log 2>&1; echo "pytest rc=$?"
grep -E "config 2:|config 3:|config 2 over|passed|failed|FAILED|XPASS" gpurun_out/s2_pytest_final.log | tail -10
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/s2_bench_final_cfg3.log 2>&1; echo "bench3 rc=$?"; tail -1 gpurun_out/s2_bench_final_cfg3.log | cut -c1-500
python bench.py --cfg 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s2_bench_final_cfg2.log 2>&1; echo "bench2 rc=$?"; tail -1 gpurun_out/s2_bench_final_cfg2.log | cut -c1-300
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s2_bench_final_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/s2_bench_final_ref.log | cut -c1-300
