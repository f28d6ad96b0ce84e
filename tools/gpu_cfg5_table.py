"""Config 5 (row a8) and the paper's preconditioner comparison (row f3, I_G / I_BD / I_pA,
P:1628-1707) on one GPU at reduced N: 3D uniform [0,1)^3, 1/r, A_ii = 100, leaf 128, NNCA
tol-1e-10 H2 matvec, GMRES(30) to 1e-10.  For eps_A in {1e-3 (BASELINE), 1e-5 (the paper's
Exp. 5 value)}: factor time, the preconditioner's own relative residual
||A M^-1 b - b|| / ||b|| (direct sum on 4096 rows, aifmm_residual), GMRES iterations with the
AIFMM preconditioner; and once per N the unpreconditioned and block-diagonal runs.
Usage: python tools/gpu_cfg5_table.py N [maxit] [eps,eps,...]   (one JSON line per run)"""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2301_12704_b200 import aifmm as A, workloads as W
cfg = W.CONFIGS[4]
n = int(sys.argv[1])
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 300
pts, b = W.make(cfg, n=n)
P = torch.from_numpy(pts).cuda()
B = torch.from_numpy(np.ascontiguousarray(b[:, 0])).cuda()
rows = W.residual_rows(n, cfg.seed)
def t(): torch.cuda.synchronize(); return time.time()
epss = [float(e) for e in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1e-3, 1e-5]
for eps in epss:
    A.free()
    t0 = t(); A.build(P, cfg.kernel_id, cfg.kparams, cfg.leaf_size, eps); t1 = t()
    A.factor(); t2 = t()
    x = A.solve(B)
    pres = A.residual(x, B, rows)
    A.matvec_build(1e-10); t3 = t()
    out = {"n": n, "eps": eps, "build_s": t1 - t0, "factor_s": t2 - t1, "matvec_build_s": t3 - t2,
           "precond_rel_residual": pres, "max_rank": A.stats()["max_rank"], "device_gb": A.stats()["device_bytes"] / 1e9}
    runs = [("pA", 1)] + ([("BD", 2), ("G", 0)] if eps == 1e-3 else [])
    for name, pre in runs:
        t4 = t(); xg, it, rr = A.gmres(B, restart=30, rtol=1e-10, maxit=maxit, precond=pre); t5 = t()
        out[f"I_{name}"] = it
        out[f"relres_{name}"] = rr
        out[f"gmres_s_{name}"] = t5 - t4
        out[f"exact_relres_{name}"] = A.residual(xg, B, rows)
    print(json.dumps(out), flush=True)
A.free()
