#!/bin/bash
# residual and largest pivot-inverse entries of config 2 under the debug toggles that used to
# move the residual (independent U/V sides vs the symmetric reading R27)
for env in "X=1" "AIFMM_NO_TSQR=1" "AIFMM_TSQR_MMAX=100000" "AIFMM_HH_CLUSTER=1" "AIFMM_ASYMMETRIC=1"; do
  echo "== $env"
  env $env AIFMM_DEBUG_PIVOTS=1 timeout 600 python tools/gpu_perf.py 1 > /tmp/pd.log 2>&1
  grep -E "aifmm pivots" /tmp/pd.log | sort -g -k13 | tail -3
  grep -E "^\{|residual" /tmp/pd.log | tail -2 | cut -c1-160
done
