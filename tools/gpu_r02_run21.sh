#!/bin/bash
set -x
python -m pytest tests -m gpu -q -rA > gpurun_out/r02_pytest_gpu21.log 2>&1; echo "pytest rc=$?"
grep -E "config 3:|N=|GMRES iter|passed|failed|FAILED" gpurun_out/r02_pytest_gpu21.log | tail -10
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
