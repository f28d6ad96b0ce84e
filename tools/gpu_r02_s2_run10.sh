#!/bin/bash
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_h2.py -q -x > gpurun_out/s2_pytest_copy.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s2_pytest_copy.log
python tools/gpu_perf.py 2 2>&1 | grep "^{" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3 build', round(d['build_s'],3), 'factor', round(d['factor_s'],3), 'res', d['residual'])"
python tools/gpu_perf.py 1 2>&1 | grep "^{" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2 build', round(d['build_s'],4), 'factor', round(d['factor_s'],4), 'res', d['residual'])"
