#!/bin/bash
# GPU tests, clean per-config timings, bench line, and the ncu evidence for profiles/:
# launch list of the bench command and a full capture of the Schur GEMM launches (NVTX "schur")
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 300 python tools/gpu_perf.py 1 > gpurun_out/perf_cfg2.log 2>&1; echo cfg2 rc=$?
timeout 600 python tools/gpu_perf.py 2 > gpurun_out/perf_cfg3.log 2>&1; echo cfg3 rc=$?
python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1; echo ncu1 rc=$?
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "schur/" -c 40 \
  -o /tmp/prof_schur -f timeout 600 python tools/gpu_perf.py 1 > gpurun_out/ncu2.log 2>&1; echo ncu2 rc=$?
python tools/ncu_kernel_traffic.py /tmp/prof_schur.ncu-rep gpurun_out/schur_ncu.json "gemm_tasks_kernel" > /dev/null 2>&1; echo summ rc=$?
ls -la /tmp/prof_schur.ncu-rep
sz=$(stat -c %s /tmp/prof_schur.ncu-rep 2>/dev/null || echo 0)
if [ "$sz" -lt 40000000 ]; then cp /tmp/prof_schur.ncu-rep gpurun_out/; fi
