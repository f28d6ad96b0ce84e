"""Build + factor + solve one config; print factor time, per-phase device ms and a hash of the
solution bytes (bitwise comparisons of kernel variants selected by environment toggles).
Usage: python tools/gpu_xhash.py <config index> [reps]"""
import sys, time, json, hashlib
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2301_12704_b200 import aifmm as A, workloads as W
cfg = W.CONFIGS[int(sys.argv[1])]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
pts, b = W.make(cfg)
P = torch.from_numpy(pts).cuda(); B = torch.from_numpy(np.ascontiguousarray(b)).cuda()
for rep in range(reps):
    A.free(); A.reset_counters(); A.set_timing(True)
    torch.cuda.synchronize(); t0 = time.time()
    A.build(P, cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol); torch.cuda.synchronize(); t1 = time.time()
    A.factor(); torch.cuda.synchronize(); t2 = time.time()
    X = A.solve(B); torch.cuda.synchronize()
    st = A.stats()
    h = hashlib.sha1(X.cpu().numpy().tobytes()).hexdigest()[:16]
    print(json.dumps({"cfg": cfg.name, "build_s": round(t1 - t0, 4), "factor_s": round(t2 - t1, 4), "xhash": h,
                      **{k: round(st[k], 2) for k in ("tri_ms", "pqr_ms", "schur_ms", "pivot_ms")}}), flush=True)
