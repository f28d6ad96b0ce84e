"""Row f2: Algorithm 2 (compress on creation) vs Algorithm 3 (deferred)
on the GPU: factor time, number of compressions, sampled direct-sum residual, max rank.
Usage: python tools/gpu_alg2.py <config index 0-4> [n]  (one JSON line per algorithm)"""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2301_12704_b200 import aifmm as A, workloads as W
cfg = W.CONFIGS[int(sys.argv[1])]
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
pts, b = W.make(cfg, n=n)
P = torch.from_numpy(pts).cuda(); B = torch.from_numpy(np.ascontiguousarray(b)).cuda()
rows = W.residual_rows(len(pts), cfg.seed)
for alg in (3, 2, 3, 2):
    A.free(); A.set_algorithm(alg); A.reset_counters(); A.set_timing(True)
    A.build(P, cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol)
    torch.cuda.synchronize(); t0 = time.time()
    A.factor(); torch.cuda.synchronize(); t1 = time.time()
    X = A.solve(B)
    st = A.stats()
    print(json.dumps({"cfg": cfg.name, "n": len(pts), "algorithm": alg, "factor_s": t1 - t0,
                      "compressions": st["compressions"], "max_rank": st["max_rank"], "top_size": st["top_size"],
                      "residual": A.residual(X, B, rows), "tri_ms": st["tri_ms"], "pqr_ms": st["pqr_ms"],
                      "redir_ms": st["redir_ms"], "schur_ms": st["schur_ms"]}), flush=True)
A.set_algorithm(3)
