#!/bin/bash
for env in "X=1" "AIFMM_MANY=100000" "AIFMM_MANY=1" "AIFMM_MANY=100000 AIFMM_PQR_MANY_MMAX=0" "AIFMM_HH_CLUSTER=1"; do
  env $env timeout 600 python tools/gpu_perf.py 1 2>/dev/null | grep '^{' | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$env', 'factor', round(d['factor_s'],3), 'res', d['residual'])"
done
