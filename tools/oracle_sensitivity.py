"""Rounding sensitivity of the oracle itself on BASELINE config 2 (full size), written to
tests/golden/cfg2_oracle_rounding_sensitivity.json.  Calls only oracle/ and the seeded input
generators (no CUDA path).

Runs of the oracle that differ only in how steps that are exact in exact arithmetic are
rounded, each compared with the reference run:
  * lu_solve: the pivot inverse P_i^{-1} (reading R16) as an LU solve against the identity
    (getrf + getrs) instead of numpy.linalg.inv (getrf + getri);
  * qr_reversed_rows: every Householder QR (the R of W^T in the two-stage RRQR, R8b, and the
    level-start orthonormalisation, R13) applied to the row-reversed matrix -- the same R (up to
    row signs) and the same Q up to the permutation, rounded along another reflector sequence;
  * both at once;
  * the compression threshold tol_c * ||F||_F (R8) scaled by (1 +- 1e-12) and (1 +- 1e-9): a
    truncation decision that sits within rounding distance of the threshold flips, as it does
    under any change of reduction order;
  * exact-arithmetic-equivalent choices of the kind a GPU implementation makes: CholeskyQR2 for
    the level-start orthonormalisation, a TSQR R factor (row chunks of <= 512 rows, R of the
    stacked chunk R's) for the first RRQR stage, Gauss-Jordan with partial pivoting for the
    pivot inverses (written here in numpy; the CUDA path is not used).
Their relative 2-norm solution differences are the method's own sensitivity to the rounding of
single steps -- the floor below which no implementation (GPU or CPU) can be compared with the
oracle (reading R24); the test bar uses the largest."""
import json
import os
import sys
import time

import numpy as np
import scipy.linalg as sl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle.factor as F                         # noqa: E402
from paper_2301_12704_b200 import workloads as W  # noqa: E402

_inv, _qr = np.linalg.inv, np.linalg.qr


def inv_lu(P):
    return sl.lu_solve(sl.lu_factor(P), np.eye(P.shape[0]))


def qr_reversed(A, mode="reduced"):
    if mode == "r":
        return _qr(A[::-1], mode="r")
    Q, R = _qr(A[::-1], mode=mode)
    return Q[::-1], R


def cholqr2(A):
    R1 = np.linalg.cholesky(A.T @ A).T
    Q1 = sl.solve_triangular(R1, A.T, trans="T").T
    R2 = np.linalg.cholesky(Q1.T @ Q1).T
    Q = sl.solve_triangular(R2, Q1.T, trans="T").T
    return Q, R2 @ R1


def tsqr_r(A, rows=512):
    n, m = A.shape
    if n <= rows or m == 0:
        return _qr(A, mode="r")
    k = -(-n // rows)
    parts = np.array_split(A, k, axis=0)
    Rs = [_qr(P, mode="r") for P in parts]
    S = np.concatenate(Rs, axis=0)
    return tsqr_r(S, rows) if S.shape[0] < n else _qr(S, mode="r")


def qr_gpu_like(A, mode="reduced"):
    if mode == "r":
        return tsqr_r(A)
    try:
        return cholqr2(A)
    except np.linalg.LinAlgError:
        return _qr(A, mode=mode)


def inv_gauss_jordan(P):
    n = P.shape[0]
    A = np.concatenate([P.astype(float), np.eye(n)], axis=1)
    for j in range(n):
        p = j + int(np.argmax(np.abs(A[j:, j])))
        if p != j:
            A[[j, p]] = A[[p, j]]
        A[j] /= A[j, j]
        col = A[:, j].copy()
        col[j] = 0.0
        A -= np.outer(col, A[j])
    return A[:, n:]


def run(cfg, pts, b, inv=None, qr=None, tol_c=None):
    np.linalg.inv = inv or _inv
    np.linalg.qr = qr or _qr
    try:
        o = F.AIFMM(pts, cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol, tol_c=tol_c).factor()
        return o, o.solve(b)
    finally:
        np.linalg.inv, np.linalg.qr = _inv, _qr


def main():
    cfg = W.CONFIGS[1]
    pts, b = W.make(cfg)
    t0 = time.time()
    o1, x1 = run(cfg, pts, b)
    out = {"workload": cfg.name, "tol": cfg.tol, "rel_solution_diff": {}, "final_rank_mismatches_per_level": {}}
    for name, kw in (("lu_solve", {"inv": inv_lu}), ("qr_reversed_rows", {"qr": qr_reversed}),
                     ("lu_solve+qr_reversed_rows", {"inv": inv_lu, "qr": qr_reversed}),
                     ("gpu_like_choices", {"inv": inv_gauss_jordan, "qr": qr_gpu_like}),
                     ("tol_c*(1+1e-12)", {"tol_c": cfg.tol * (1 + 1e-12)}),
                     ("tol_c*(1-1e-12)", {"tol_c": cfg.tol * (1 - 1e-12)}),
                     ("tol_c*(1+1e-9)", {"tol_c": cfg.tol * (1 + 1e-9)}),
                     ("tol_c*(1-1e-9)", {"tol_c": cfg.tol * (1 - 1e-9)})):
        o2, x2 = run(cfg, pts, b, **kw)
        out["rel_solution_diff"][name] = float(np.linalg.norm(x2 - x1) / np.linalg.norm(x1))
        out["final_rank_mismatches_per_level"][name] = {
            str(l): int(sum(1 for bx in o1.levels[l].boxes if o1.levels[l].k[bx] != o2.levels[l].k[bx])) for l in o1.levels}
        print(name, out["rel_solution_diff"][name], flush=True)
    out["rel_solution_diff_inv_vs_lu_solve"] = out["rel_solution_diff"]["lu_solve"]
    out["rel_solution_diff_max"] = max(out["rel_solution_diff"].values())
    out["seconds"] = time.time() - t0
    out["script"] = "tools/oracle_sensitivity.py"
    path = os.path.join(ROOT, "tests", "golden", "cfg2_oracle_rounding_sensitivity.json")
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
