"""Dense references (oracle; test infrastructure only).

* dense_matrix: A_ij = K(x_i, x_j) written out, user order.
* h2_matrix: the NNCA approximation of A (Eq. NCA P:347-357 with the nested operators of
  P:360-367 and Table) written out densely, user order: near leaf pairs exact,
  every IL pair (B, D) at level l replaced by U_B^full A(sk B, sk D) V_D^full^*.
* residual: ||A x - b|| / ||b|| by exact direct sum on (a sample of) rows.
"""
from __future__ import annotations

import numpy as np

from . import kernels


def dense_matrix(points, kernel_id, kparams):
    n = points.shape[0]
    idx = np.arange(n)
    return kernels.entries(kernel_id, kparams, points, points, idx, idx)


def full_bases(aifmm):
    """U^full[l][B]: (|points(B)| x k_B), nested through the NNCA operators (V = U, R10)."""
    t, nn = aifmm.tree, aifmm.nnca
    Uf = {t.L: {B: nn.U[t.L][B] for B in nn.U[t.L]}}
    for l in range(t.L - 1, 1, -1):
        Uf[l] = {}
        for B in nn.U[l]:
            rows = nn.child_rows(l, B)
            parts = [Uf[l + 1][c] @ nn.U[l][B][r0:r1] for c, (r0, r1) in rows.items()]
            Uf[l][B] = np.concatenate(parts, axis=0) if parts else np.zeros((0, nn.rank(l, B)))
    return Uf


def h2_matrix(aifmm):
    """Densified NNCA matrix in user order."""
    t, nn = aifmm.tree, aifmm.nnca
    n = t.n
    M = np.full((n, n), np.nan)
    pts = t.points
    Uf = full_bases(aifmm)
    for l in range(2, t.L + 1):
        for B in aifmm.il[l]:
            a0, a1 = t.point_range(l, B)
            for D in aifmm.il[l][B]:
                b0, b1 = t.point_range(l, D)
                Abd = kernels.block(aifmm.kid, aifmm.kp, pts, nn.sk[l][B], nn.sk[l][D])
                M[a0:a1, b0:b1] = Uf[l][B] @ Abd @ Uf[l][D].T
    L = t.L
    for B in aifmm.near[L]:
        a0, a1 = t.point_range(L, B)
        for D in aifmm.near[L][B]:
            b0, b1 = t.point_range(L, D)
            M[a0:a1, b0:b1] = kernels.block(aifmm.kid, aifmm.kp, pts, np.arange(a0, a1), np.arange(b0, b1))
    assert not np.isnan(M).any(), "NNCA blocks do not cover the matrix"
    out = np.empty_like(M)
    out[np.ix_(t.perm, t.perm)] = M
    return out


def far_block_errors(aifmm):
    """Relative Frobenius error of every IL block at every level vs the dense block."""
    t, nn = aifmm.tree, aifmm.nnca
    Uf = full_bases(aifmm)
    errs = []
    for l in range(2, t.L + 1):
        for B in aifmm.il[l]:
            a0, a1 = t.point_range(l, B)
            for D in aifmm.il[l][B]:
                b0, b1 = t.point_range(l, D)
                ex = kernels.block(aifmm.kid, aifmm.kp, t.points, np.arange(a0, a1), np.arange(b0, b1))
                Abd = kernels.block(aifmm.kid, aifmm.kp, t.points, nn.sk[l][B], nn.sk[l][D])
                ap = Uf[l][B] @ Abd @ Uf[l][D].T
                errs.append((l, B, D, np.linalg.norm(ap - ex) / np.linalg.norm(ex)))
    return errs


def residual(points, kernel_id, kparams, x, b, rows=None):
    """||A x - b||_2 / ||b||_2 over `rows` (all rows if None), exact direct sum."""
    n = points.shape[0]
    rows = np.arange(n) if rows is None else np.asarray(rows)
    x2 = x if x.ndim == 2 else x[:, None]
    b2 = b if b.ndim == 2 else b[:, None]
    r2 = 0.0
    for s in range(0, rows.size, 256):
        rr = rows[s:s + 256]
        A = kernels.entries(kernel_id, kparams, points[rr], points, rr, np.arange(n))
        r2 += np.sum((A @ x2 - b2[rr]) ** 2)
    return float(np.sqrt(r2) / np.linalg.norm(b2[rows]))
