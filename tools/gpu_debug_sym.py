"""Debug: GPU vs the C++ oracle on the config-1 grid case under the R30 / R31 toggles."""
import sys, os, subprocess, json
sys.path.insert(0, '.')
code = r'''
import sys, os; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2301_12704_b200 import aifmm as A, workloads as W
from oracle.cpp import CppAIFMM
pts = W.make_points("grid", 4096, 2, 21); b = W.make_rhs(4096, 1, 21)
xo = CppAIFMM(pts, 0, (10.0, 0.0), 64, 1e-8).factor().solve(b)
A.build(torch.from_numpy(pts).cuda(), 0, (10.0, 0.0), 64, 1e-8); A.factor()
x = A.solve(torch.from_numpy(b).cuda()).cpu().numpy()
print("REL", np.linalg.norm(x - xo) / np.linalg.norm(xo))
'''
for env in ({}, {"AIFMM_NO_SYM_SCHUR": "1"}, {"AIFMM_NO_NULLSPACE": "1"}, {"AIFMM_NO_SYM_SCHUR": "1", "AIFMM_NO_NULLSPACE": "1"}, {"AIFMM_DEBUG_SYM": "1"}):
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True, timeout=600)
    print(env, [l for l in r.stdout.splitlines() if "REL" in l], r.stderr[-3000:] if ("DEBUG" in str(env) or r.returncode) else "")
