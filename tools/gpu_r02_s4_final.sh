#!/bin/bash
# session-4 final evidence on the last build: config-2 bench line, reference arm, launch list of
# the bench command, ncu --set full of the Schur DMMA GEMM (traffic figure for bench.py's roofline)
python bench.py --cfg 2 --no-cpu-baseline > gpurun_out/s4_bench_cfg2.log 2>&1; echo "bench2 rc=$?"
timeout 400 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/s4_bench_ref.log 2>&1; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4_launches_cfg3.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/s4_ncu_launches.log 2>&1; echo "ncu list rc=$?"
python tools/ncu_summary.py gpurun_out/s4_launches_cfg3.csv > gpurun_out/s4_launches_cfg3_summary.txt 2>&1; head -25 gpurun_out/s4_launches_cfg3_summary.txt
rm -f gpurun_out/s4_launches_cfg3.csv
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "schur/" --launch-skip 4 -c 8 -o /tmp/prof_schur4 -f \
  python tools/gpu_once.py 2 > gpurun_out/s4_ncu_schur.log 2>&1; echo "ncu schur rc=$?"
python tools/ncu_kernel_traffic.py /tmp/prof_schur4.ncu-rep gpurun_out/s4_schur_gemm_ncu_cfg3.json "gemm_tasks_kernel" > /dev/null 2>&1
cat gpurun_out/s4_schur_gemm_ncu_cfg3.json
