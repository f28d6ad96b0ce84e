#!/bin/bash
# session 3: split hh_update default -- seg sweep (bitwise), GPU suite with the hard config-2
# gate, config-3 bench line, launch list and ncu --set full of the two trailing-update passes
for sg in 128 256; do AIFMM_HHU_SEG=$sg python tools/gpu_xhash.py 2 2 | tail -1 | sed "s/^/seg$sg /"; done
python -m pytest tests -m gpu -q -rA > gpurun_out/s3_pytest2.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|XPASS|Error" gpurun_out/s3_pytest2.log | tail -6; grep "config 2:" gpurun_out/s3_pytest2.log | head -1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/s3_bench_cfg3.log 2>&1; echo "bench3 rc=$?"; tail -1 gpurun_out/s3_bench_cfg3.log | cut -c1-400
python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/s3_bench_plain.log 2>&1; echo "plain rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3_launches_cfg3.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/s3_ncu_launches.log 2>&1; echo "ncu list rc=$?"
python tools/ncu_summary.py gpurun_out/s3_launches_cfg3.csv > gpurun_out/s3_launches_cfg3_summary.txt 2>&1; head -16 gpurun_out/s3_launches_cfg3_summary.txt
rm -f gpurun_out/s3_launches_cfg3.csv
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:hh_update --launch-skip 200 -c 8 -o gpurun_out/prof_hhu3 -f \
  python tools/gpu_once.py 2 > gpurun_out/s3_ncu_hhu.log 2>&1; echo "ncu hhu rc=$?"
python tools/ncu_kernel_traffic.py gpurun_out/prof_hhu3.ncu-rep gpurun_out/s3_hhu_ncu_cfg3.json "hh_update" > /dev/null 2>&1; head -30 gpurun_out/s3_hhu_ncu_cfg3.json
