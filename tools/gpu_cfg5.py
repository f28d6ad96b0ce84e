"""Config 5 (row a8) on one GPU: AIFMM factor at tol 1e-3 as right preconditioner of
GMRES(30) with the NNCA tol-1e-10 H2 matvec, stop at relative residual 1e-10.  Optional N
(default: the full 2^21 points of BASELINE config 5; BASELINE shards that over 8 GPUs)."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2301_12704_b200 import aifmm as A, workloads as W
cfg = W.CONFIGS[4]
n = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.n
pts, b = W.make(cfg, n=n)
P = torch.from_numpy(pts).cuda()
B = torch.from_numpy(np.ascontiguousarray(b[:, 0])).cuda()
out = {"cfg": cfg.name, "n": n}
def t(): torch.cuda.synchronize(); return time.time()
t0 = t(); A.build(P, cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol); t1 = t()
A.factor(); t2 = t()
A.matvec_build(1e-10); t3 = t()
x, it, rr = A.gmres(B, restart=30, rtol=1e-10, maxit=300, precond=True); t4 = t()
out.update(build_s=t1 - t0, factor_s=t2 - t1, matvec_build_s=t3 - t2, gmres_s=t4 - t3, iterations=it, relres_h2=rr)
st = A.stats(); out["device_gb"] = st["device_bytes"] / 1e9; out["max_rank"] = st["max_rank"]
print(json.dumps(out), flush=True)
if len(sys.argv) > 2:
    from oracle import dense
    rows = W.residual_rows(n, cfg.seed)
    out["relres_exact_4096rows"] = dense.residual(pts, cfg.kernel_id, cfg.kparams, x.cpu().numpy(), b[:, 0], rows)
    print(json.dumps(out), flush=True)
