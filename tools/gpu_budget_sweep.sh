#!/bin/bash
for v in "48 48" "32 24" "24 48"; do set -- $v
  AIFMM_CMP_BUDGET_GB=$1 AIFMM_ACA_BUDGET_GB=$2 python tools/gpu_perf.py 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cmp $1 aca $2', 'build', round(d['build_s'],3), 'factor', round(d['factor_s'],3), 'GB', round(d['device_bytes']/1e9,1), 'syncs', d['host_syncs'], 'res', d['residual'])"
done
for v in "6 6" "24 24" "48 48"; do set -- $v
  AIFMM_CMP_BUDGET_GB=$1 AIFMM_ACA_BUDGET_GB=$2 python tools/gpu_perf.py 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2 cmp $1 aca $2', 'build', round(d['build_s'],4), 'factor', round(d['factor_s'],4), 'GB', round(d['device_bytes']/1e9,2), 'syncs', d['host_syncs'], 'res', d['residual'])"
done
