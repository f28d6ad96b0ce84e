#!/bin/bash
# config-3 factor time under routing toggles, with the 48 GB batch budget
for env in "X=1" "AIFMM_MANY=48" "AIFMM_MANY=192" "AIFMM_PQR_MANY_MMAX=1100" "AIFMM_PQR_MANY_MMAX=400" "AIFMM_NULLSPACE=1" "AIFMM_NULLSPACE_PMAX=128" "AIFMM_GEMM_WIDE=1" "AIFMM_TSQR_ROWS=2048" "AIFMM_REGCL_FEW=1" "X=2"; do
  env $env timeout 600 python tools/gpu_perf.py 2 2>/dev/null | grep '^{' | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$env', 'build', round(d['build_s'],3), 'factor', round(d['factor_s'],3), 'res', d['residual'], 'tri', round(d['tri_ms']), 'pqr', round(d['pqr_ms']), 'piv', round(d['pivot_ms']))"
done
