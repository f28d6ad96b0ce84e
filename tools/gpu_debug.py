"""GPU vs oracle step-by-step comparison on small problems (debug aid, not a test)."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2301_12704_b200 import aifmm as A, workloads as W
from oracle.factor import AIFMM
from oracle import dense

def run(pts, b, kid, kp, leaf, tol, tol_c=None, label=""):
    d = pts.shape[1]
    t0 = time.time()
    o = AIFMM(pts, kid, kp, leaf, tol, tol_c=tol_c).factor()
    xo = o.solve(b)
    to = time.time() - t0
    A.free()
    if tol_c is not None:
        A.set_compression_tol(tol_c)
    A.build(torch.from_numpy(pts).cuda(), kid, kp, leaf, tol)
    perm, L = A.get_tree(len(pts))
    res = {"label": label, "L": (L, o.tree.L), "perm": bool(np.array_equal(perm, o.tree.perm))}
    ok_lists = True; ok_col = True; ok_rank = True; rk = []
    for l in range(2, L + 1):
        off = A.get_level_offsets(l, d)
        ok_lists &= bool(np.array_equal(off, o.tree.off[l]))
        nptr, nidx, iptr, iidx = A.get_lists(l, d)
        col = A.get_colours(l, d)
        r = A.get_ranks(l, d, 0)
        for bx in o.near[l]:
            ok_lists &= list(nidx[nptr[bx]:nptr[bx+1]]) == o.near[l][bx]
            ok_lists &= list(iidx[iptr[bx]:iptr[bx+1]]) == o.il[l][bx]
            ok_col &= int(col[bx]) == o.colour[l][bx]
            if int(r[bx]) != o.nnca.rank(l, bx):
                ok_rank = False; rk.append((l, bx, int(r[bx]), o.nnca.rank(l, bx)))
    res.update(lists=ok_lists, colours=ok_col, nnca_ranks=ok_rank, rank_mismatch=rk[:5])
    torch.cuda.synchronize()
    A.factor()
    fr_ok = True
    for l in range(2, L + 1):
        r = A.get_ranks(l, d, 1)
        for bx in o.near[l]:
            if int(r[bx]) != o.levels[l].k[bx]:
                fr_ok = False
    res["final_ranks"] = fr_ok
    X = A.solve(torch.from_numpy(b).cuda()).cpu().numpy()
    res["rel_diff_vs_oracle"] = float(np.linalg.norm(X - xo) / np.linalg.norm(xo))
    res["res_gpu"] = dense.residual(pts, kid, kp, X, b, W.residual_rows(len(pts), 0))
    res["res_oracle"] = dense.residual(pts, kid, kp, xo, b, W.residual_rows(len(pts), 0))
    res["oracle_s"] = to
    res["stats"] = A.stats()
    print(json.dumps(res), flush=True)

if __name__ == "__main__":
    pts, b = W.small_problem(d=2, n=2048, seed=3)
    run(pts, b, 2, (float(np.sqrt(1000*2048)), 0.0), 32, 1e-8, label="rand2d_invr")
    cfg = W.CONFIGS[0]; pts, b = W.make(cfg)
    run(pts, b, cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol, label="cfg1")
    pts, b = W.small_problem(d=2, n=3000, seed=4, nrhs=3)
    run(pts, b, 1, (1.01, 0.1), 24, 1e-6, label="rand2d_exp")
    run(pts, b, 0, (10.0, 0.0), 24, 1e-5, tol_c=0.0, label="exact")
    pts, b = W.small_problem(d=3, n=3000, kind="uniform_01", seed=5)
    run(pts, b, 2, (100.0, 0.0), 32, 1e-6, label="3d")
