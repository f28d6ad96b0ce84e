cd $GRAFT_REPO_ROOT
for ph in 1 2 4 7; do echo "phases $ph:"; AIFMM_DIST_PHASES=$ph timeout 300 python tools/gpu_dist_debug.py 2 12000 2 2>&1 | tail -1; done
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -rA -x -s > gpurun_out/s2_pytest_dist.log 2>&1; echo "pytest dist rc=$?"
grep -E "world|passed|failed|FAILED|Error|error" gpurun_out/s2_pytest_dist.log | tail -20
