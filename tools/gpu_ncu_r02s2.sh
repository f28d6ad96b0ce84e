#!/bin/bash
# session-2 evidence: config-3 bench launch list (after a clean run of the same command) and an
# ncu --set full capture of the changed Gauss-Jordan panel kernel (level-5/6 pivots)
python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/s2_bench_plain.log 2>&1; echo "plain rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2_launches_cfg3.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/s2_ncu_launches.log 2>&1; echo "ncu list rc=$?"
python tools/ncu_summary.py gpurun_out/s2_launches_cfg3.csv > gpurun_out/s2_launches_cfg3_summary.txt 2>&1; head -16 gpurun_out/s2_launches_cfg3_summary.txt
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gj_panel_kernel --launch-skip 60 -c 6 -o /tmp/prof_gj2 -f \
  python tools/gpu_once.py 2 > gpurun_out/s2_ncu_gj.log 2>&1; echo "ncu gj rc=$?"
python tools/ncu_kernel_traffic.py /tmp/prof_gj2.ncu-rep gpurun_out/s2_gj_ncu_cfg3.json "gj_" > /dev/null 2>&1; cat gpurun_out/s2_gj_ncu_cfg3.json | head -20
