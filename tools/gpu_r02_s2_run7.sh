#!/bin/bash
timeout 1200 python -m pytest tests/test_gpu_dist.py -q -x -s > gpurun_out/s2_pytest_dist3.log 2>&1; echo "dist rc=$?"; grep -E "world|passed|failed" gpurun_out/s2_pytest_dist3.log | tail -6
AIFMM_DIST_FORCE=1 timeout 1200 python tools/gpu_dist_scaling.py 1 > gpurun_out/s2_dist_scaling_cfg2.jsonl 2> gpurun_out/s2_dist_scaling_cfg2.err; echo "scaling rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/s2_dist_scaling_cfg2.jsonl"):
    d = json.loads(l)
    print(d["world"], d["replicas_bitwise_identical"], {k: round(d[k]["imbalance"], 2) for k in ("schur_flops", "pivot_flops", "tri_flops", "mult_flops")}, max(d["exchange_gb_received_per_rank"]))
PY
bash tools/gpu_aca_sweep.sh
