#!/bin/bash
# session-3 health check: GPU suite, smoke, config-3 bench line
python -m pytest tests -m gpu -q -rA > gpurun_out/s3_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|XPASS|error" gpurun_out/s3_pytest.log | tail -10
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/s3_bench_cfg3.log 2>&1; echo "bench3 rc=$?"; tail -1 gpurun_out/s3_bench_cfg3.log | cut -c1-600
