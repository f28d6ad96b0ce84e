"""The rounding floor of BASELINE config 2 (N = 65536, log r, tol 1e-10): how far apart two
correct FP64 evaluations of the SAME AIFMM (identical integer decisions) land.

Run A: the numpy oracle as it stands (pivot inverses by numpy.linalg.inv, reading R16), with
every decision of the truncated pivoted QR (R7 pivot index, R8 discard flag, truncation rank)
recorded.  Run B: the same oracle with the pivot inverses computed by an LU solve against the
identity (scipy lu_factor + lu_solve; exact-arithmetic-equivalent), REPLAYING run A's
decisions (same pivots, same ranks in every box -- checked).  NNCA decisions are identical
anyway (ACA on exact kernel entries).  The relative 2-norm difference of the two solutions is
pure rounding propagation: no implementation, CPU or GPU, can be compared with the oracle
more tightly than this on this workload.  A third run C (LU-solve inverses, free decisions)
shows how much the decisions themselves add.

Calls only oracle/ and the seeded input generators.  Writes
tests/golden/cfg2_oracle_rounding_floor.json."""
import json
import os
import sys
import time

import numpy as np
import scipy.linalg as sl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle.factor as F                          # noqa: E402
from oracle import dense                           # noqa: E402
from oracle.linalg import pick                     # noqa: E402
from paper_2301_12704_b200 import workloads as W   # noqa: E402

_inv = np.linalg.inv
_pqe = F.pivoted_qr_extend


def inv_lu(P):
    return sl.lu_solve(sl.lu_factor(P), np.eye(P.shape[0]))


def make_pqe(mode, log):
    """oracle/linalg.py: pivoted_qr_extend with its decisions recorded (mode 'record') or
    replayed from `log` (mode 'replay'); the arithmetic is the same."""
    ctr = [0]

    def pqe(W_, basis, tau, tmin, tmax):
        W_ = np.array(W_, dtype=np.float64, copy=True)
        m = W_.shape[0]
        B = basis.copy() if basis is not None else np.zeros((m, 0))
        seq, t_rec = (log[ctr[0]] if mode == "replay" else ([], None))
        ctr[0] += 1
        qs, t_trunc, step = [], None, 0
        while len(qs) < tmax:
            norms2 = np.sum(W_ * W_, axis=0) if W_.shape[1] else np.zeros(0)
            res = np.sqrt(np.sum(norms2))
            if mode == "replay":
                if step >= len(seq):
                    break
                j, disc = seq[step]
            else:
                if t_trunc is None and not res > tau:
                    t_trunc = len(qs)
                if len(qs) >= tmin and not res > tau:
                    break
                j = pick(np.sqrt(norms2))
                if j is None:
                    break
            step += 1
            w = W_[:, j].copy()
            w = w - B @ (B.T @ w)
            n1 = np.linalg.norm(w)
            w = w - B @ (B.T @ w)
            nw = np.linalg.norm(w)
            if not nw > 0.5 * n1:
                n2 = nw
                w = w - B @ (B.T @ w)
                nw = np.linalg.norm(w)
                if not nw > 0.5 * n2:
                    nw = 0.0
            if mode == "replay":
                if disc:
                    nw = 0.0
                elif not nw > 0.0:
                    raise RuntimeError("replayed pivot collapsed")
            else:
                seq.append((j, not nw > 0.0))
            if not nw > 0.0:
                W_[:, j] = 0.0
                continue
            q = w / nw
            qs.append(q)
            B = np.concatenate([B, q[:, None]], axis=1)
            W_ = W_ - np.outer(q, q @ W_)
            W_[:, j] = 0.0
        if mode == "replay":
            t_trunc = t_rec
        else:
            if t_trunc is None:
                t_trunc = len(qs)
            log.append((seq, t_trunc))
        Q = np.stack(qs, axis=1) if qs else np.zeros((m, 0))
        return Q, t_trunc
    return pqe


def run(cfg, pts, b, inv, pqe):
    np.linalg.inv = inv
    F.pivoted_qr_extend = pqe
    try:
        o = F.AIFMM(pts, cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol).factor()
        return o, o.solve(b)
    finally:
        np.linalg.inv, F.pivoted_qr_extend = _inv, _pqe


def main():
    cfg = W.CONFIGS[1]
    pts, b = W.make(cfg)
    t0 = time.time()
    log = []
    oa, xa = run(cfg, pts, b, _inv, make_pqe("record", log))
    ob, xb = run(cfg, pts, b, inv_lu, make_pqe("replay", log))
    oc, xc = run(cfg, pts, b, inv_lu, _pqe)
    mism = lambda o1, o2: {str(l): int(sum(o1.levels[l].k[x] != o2.levels[l].k[x] for x in o1.levels[l].boxes))
                           for l in o1.levels}
    rows = W.residual_rows(cfg.n, cfg.seed)
    out = {
        "workload": cfg.name, "tol": cfg.tol,
        "same_decisions_rel_solution_diff": float(np.linalg.norm(xb - xa) / np.linalg.norm(xa)),
        "same_decisions_rank_mismatches": mism(oa, ob),
        "free_decisions_rel_solution_diff": float(np.linalg.norm(xc - xa) / np.linalg.norm(xa)),
        "free_decisions_rank_mismatches": mism(oa, oc),
        "residual_4096_rows": {"A": dense.residual(pts, cfg.kernel_id, cfg.kparams, xa, b, rows),
                               "B": dense.residual(pts, cfg.kernel_id, cfg.kparams, xb, b, rows),
                               "C": dense.residual(pts, cfg.kernel_id, cfg.kparams, xc, b, rows)},
        "decisions_recorded": len(log),
        "seconds": time.time() - t0,
        "script": "tools/oracle_decision_replay.py",
    }
    json.dump(out, open(os.path.join(ROOT, "tests", "golden", "cfg2_oracle_rounding_floor.json"), "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
