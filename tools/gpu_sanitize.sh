#!/bin/bash
# compute-sanitizer memcheck of one small build + factor + solve (+ GMRES, residual) on cuda:0
set -x
cat > /tmp/san.py <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2301_12704_b200 import aifmm as A, workloads as W
for kid, kp, d, kind in ((0, (10.0, 0.0), 2, "uniform_pm1"), (2, (100.0, 0.0), 3, "uniform_01")):
    pts, b = W.small_problem(d=d, n=3000, kind=kind, seed=3, nrhs=2)
    A.free(); A.build(torch.from_numpy(pts).cuda(), kid, kp, 40, 1e-6); A.factor()
    B = torch.from_numpy(b).cuda(); X = A.solve(B); r = A.residual(X, B)
    A.matvec_build(1e-8); x, it, rr = A.gmres(B[:, 0].contiguous(), precond=2, maxit=30)
    print("ok", kid, r, it, flush=True)
PY
timeout 1800 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python /tmp/san.py > gpurun_out/r02_memcheck.log 2>&1; echo "memcheck rc=$?"
tail -5 gpurun_out/r02_memcheck.log
