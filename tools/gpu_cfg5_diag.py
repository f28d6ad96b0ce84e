"""Config-5 pieces at a given N: factor residual, H2 matvec accuracy (sampled exact rows),
then GMRES (debug aid)."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2301_12704_b200 import aifmm as A, workloads as W
from oracle import dense, kernels
cfg = W.CONFIGS[4]
n = int(sys.argv[1])
leaf = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.leaf_size
ptol = float(sys.argv[3]) if len(sys.argv) > 3 else cfg.tol
pts, b = W.make(cfg, n=n)
b = b[:, 0]
rows = W.residual_rows(n, cfg.seed, 1024)
def exact_rows(x):
    Ar = kernels.entries(cfg.kernel_id, cfg.kparams, pts[rows], pts, rows, np.arange(n))
    return Ar @ x
P = torch.from_numpy(pts).cuda(); B = torch.from_numpy(np.ascontiguousarray(b)).cuda()
out = {"n": n, "leaf": leaf, "ptol": ptol}
t0 = time.time(); A.build(P, cfg.kernel_id, cfg.kparams, leaf, ptol); A.factor(); torch.cuda.synchronize(); out["build_factor_s"] = time.time() - t0
xf = A.solve(B).cpu().numpy()
out["factor_relres_rows"] = float(np.linalg.norm(exact_rows(xf) - b[rows]) / np.linalg.norm(b[rows]))
out["max_rank"] = A.stats()["max_rank"]
t0 = time.time(); A.matvec_build(1e-10); torch.cuda.synchronize(); out["mv_build_s"] = time.time() - t0
xr = np.random.default_rng(0).standard_normal(n)
y = A.matvec(torch.from_numpy(xr).cuda()).cpu().numpy()
ye = exact_rows(xr)
out["matvec_rel_err_rows"] = float(np.linalg.norm(y[rows] - ye) / np.linalg.norm(ye))
print(json.dumps(out), flush=True)
t0 = time.time(); x, it, rr = A.gmres(B, restart=30, rtol=1e-10, maxit=60, precond=True); torch.cuda.synchronize()
out.update(gmres_s=time.time() - t0, it=it, rr=rr)
xh = x.cpu().numpy()
out["gmres_exact_relres_rows"] = float(np.linalg.norm(exact_rows(xh) - b[rows]) / np.linalg.norm(b[rows]))
yx = A.matvec(x).cpu().numpy()
out["h2_relres_of_x"] = float(np.linalg.norm(yx - b) / np.linalg.norm(b))
out["h2_vs_exact_on_x_rows"] = float(np.linalg.norm(yx[rows] - exact_rows(xh)) / np.linalg.norm(exact_rows(xh)))
out["x_norm"] = float(np.linalg.norm(xh)); out["xf_norm"] = float(np.linalg.norm(xf))
print(json.dumps(out), flush=True)
