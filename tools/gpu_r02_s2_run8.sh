#!/bin/bash
# lazy fill-in slots: parity + memory A/B
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x > gpurun_out/s2_pytest_lazy.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s2_pytest_lazy.log
for e in lazy eager; do
  if [ $e = eager ]; then export AIFMM_EAGER_FILL=1; fi
  python tools/gpu_perf.py 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', 'factor', round(d['factor_s'],3), 'GB', round(d['device_bytes']/1e9,1), 'res', d['residual'])"
  python tools/gpu_perf.py 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e cfg2', 'factor', round(d['factor_s'],3), 'GB', round(d['device_bytes']/1e9,2), 'res', d['residual'])"
done
unset AIFMM_EAGER_FILL
AIFMM_PROFILE=1 python tools/gpu_perf.py 2 2>&1 | grep "level" | head -7 | cut -c1-250
