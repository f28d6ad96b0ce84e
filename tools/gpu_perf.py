"""Per-phase timing of build/factor/solve on a config (AIFMM_PROFILE=1 for the breakdown).
Usage: python tools/gpu_perf.py <config index 0-4> [n]  (prints one JSON line per repetition)"""
import sys, time, json, os
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2301_12704_b200 import aifmm as A, workloads as W
cfgi = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
cfg = W.CONFIGS[cfgi]
pts, b = W.make(cfg, n=n)
P = torch.from_numpy(pts).cuda(); B = torch.from_numpy(np.ascontiguousarray(b)).cuda()
rows = W.residual_rows(len(pts), cfg.seed)
for rep in range(2):
    A.free(); A.reset_counters(); A.set_timing(True)
    torch.cuda.synchronize(); t0 = time.time()
    A.build(P, cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol); torch.cuda.synchronize(); t1 = time.time()
    A.factor(); torch.cuda.synchronize(); t2 = time.time()
    X = A.solve(B); torch.cuda.synchronize(); t3 = time.time()
    st = A.stats()
    res = A.residual(X, B, rows)
    print(json.dumps({"cfg": cfg.name, "n": len(pts), "build_s": t1-t0, "factor_s": t2-t1, "solve_s": t3-t2, "residual": res,
                      **{k: st[k] for k in ("levels","top_size","max_rank","launches","host_syncs","compressions","schur_flops",
                                            "factor_flops","device_bytes","schur_ms","pivot_ms","tri_ms","pqr_ms","redir_ms",
                                            "mult_ms","proj_ms","fresh_ms","orth_ms")}}), flush=True)
