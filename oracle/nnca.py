"""NNCA: nested cross approximation of the far field (oracle; test infrastructure only).

Eq. NCA:
    A(t^X, s^Y) ~= A(t^X, s^{X,i}) A(t^{X,i}, s^{X,i})^{-1} A(t^{X,i}, s^{Y,o}) A(t^{Y,o}, s^{Y,o})^{-1} A(t^{Y,o}, s^Y)
with row pivots t^{X,i} in t^X and far pivots s^{X,i} in F^{X,i} = sources of IL(X) (Eq. Fj, P:353;
R11b: points of the IL boxes at the leaf level, their children's skeletons above).
Operators: U_B = A(t^B, s^{B,i}) A(t^{B,i}, s^{B,i})^{-1} (L2P, stacked L2L at
non-leaf levels, Table); V_B^* = A(t^{B,o}, s^{B,o})^{-1} A(t^{B,o}, s^B) (P2M / M2M);
M2L A_BD = A(t^{B,i}, s^{D,o}); near K_BX = A(t^B, s^X).

Readings: R9 the pivot rule (deferred by P:359 to another paper) is ACA with
partial pivoting on A(R_B, F_B); R10 u = v and a symmetric kernel give one skeleton
sk(B) = t^{B,i} = s^{B,o} and one far-pivot set fp(B) = s^{B,i} = t^{B,o}, so V_B = U_B;
R11 at non-leaf levels the candidate rows R_B are the children's skeletons stacked in
Morton order (Eq. P:414-416: particles of a parent are its children's multipoles); R20 when
IL(B) holds fewer points than R_B, the ancestors' interaction lists are appended to F_B.
"""
from __future__ import annotations

import numpy as np

from . import kernels
from .linalg import pick

GUARD = 1e-13      # R9: a cross whose pivot is below GUARD * max|previous pivots| is not accepted


def aca(row_fn, col_fn, nR: int, nF: int, eps: float):
    """ACA with partial pivoting (R9).

    row_fn(i) -> A(R[i], F) (length nF); col_fn(j) -> A(R, F[j]) (length nR).
    Returns (row pivots, column pivots) in pivot order.
    """
    us, vs, rp, cp = [], [], [], []
    rows_used = np.zeros(nR, dtype=bool)
    cols_used = np.zeros(nF, dtype=bool)
    kmax = min(nR, nF)
    i = 0
    norm2 = 0.0
    first = None
    while len(us) < kmax:
        rows_used[i] = True
        r = row_fn(i).astype(np.float64)
        for u, v in zip(us, vs):            # residual row, crosses in order
            r = r - u[i] * v
        j = pick(r, cols_used)
        if j is None:
            free = np.flatnonzero(~rows_used)
            if free.size == 0:
                break
            i = int(free[0])
            continue
        delta = r[j]
        if first is not None and abs(delta) <= GUARD * first:
            break
        first = abs(delta) if first is None else max(first, abs(delta))
        v = r / delta
        c = col_fn(j).astype(np.float64)
        for u, vv in zip(us, vs):
            c = c - vv[j] * u
        u = c
        cols_used[j] = True
        uu = float(u @ u)
        vv2 = float(v @ v)
        cross = 0.0
        for u0, v0 in zip(us, vs):
            cross += float(u0 @ u) * float(v0 @ v)
        norm2 = norm2 + 2.0 * cross + uu * vv2
        us.append(u)
        vs.append(v)
        rp.append(i)
        cp.append(j)
        if np.sqrt(uu * vv2) <= eps * np.sqrt(max(norm2, 0.0)):
            break
        nxt = pick(u, rows_used)
        if nxt is None:
            free = np.flatnonzero(~rows_used)
            if free.size == 0:
                break
            nxt = int(free[0])
        i = nxt
    return np.array(rp, dtype=np.int64), np.array(cp, dtype=np.int64)


class NNCA:
    """Per level l (L..2), per non-empty box B:
       R[l][B]  candidate rows (global tree-order point indices) = x-variables of B
       sk[l][B] skeleton rows (subset of R), fp[l][B] far pivots (subset of F_B)
       U[l][B]  |R| x k operator A(R, fp) A(sk, fp)^{-1}; V = U (R10)
    """

    def __init__(self, tree, near, il, kernel_id, kparams, eps):
        self.t, self.kid, self.kp = tree, kernel_id, kparams
        self.R, self.sk, self.fp, self.U = {}, {}, {}, {}
        pts = tree.points
        for l in range(tree.L, 1, -1):
            self.R[l], self.sk[l], self.fp[l], self.U[l] = {}, {}, {}, {}
            for B in sorted(near[l]):
                if l == tree.L:
                    a, b = tree.point_range(l, B)
                    self.R[l][B] = np.arange(a, b, dtype=np.int64)
                else:
                    parts = [self.sk[l + 1][c] for c in tree.children(l, B)]
                    self.R[l][B] = np.concatenate(parts) if parts else np.zeros(0, np.int64)
            for B in sorted(near[l]):
                R = self.R[l][B]
                # R11b: the sources s^{X'} of an IL box X' at level l are its x-variables, i.e.
                # its points at the leaf level and its children's skeletons above (Eq. Fj
                # with Eq. P:414-416) -- the same sets as the candidate rows R_{X'}
                F = [self.R[l][D] for D in il[l][B]]
                # R20: a sparse neighbourhood can leave IL(B) with fewer sources than R_B; then
                # the IL of the ancestors (coarser far field of B) is appended, parent first,
                # each ancestor IL box D represented by the same nested sources: its points at the
                # leaf level, else the skeletons of its level-(l+1) descendants (Morton order)
                la, A_ = l, B
                while sum(f.size for f in F) < R.size and la > 2:
                    la, A_ = la - 1, A_ >> tree.d
                    for D in il[la][A_]:
                        if l == tree.L:
                            F.append(np.arange(*tree.point_range(la, D), dtype=np.int64))
                        else:
                            sh = tree.d * (l + 1 - la)
                            F += [self.sk[l + 1][c] for c in range(D << sh, (D + 1) << sh)
                                  if c in self.sk[l + 1]]
                F = np.concatenate(F) if F else np.zeros(0, np.int64)
                self.R[l][B] = R
                if R.size == 0 or F.size == 0:
                    ri = np.zeros(0, np.int64)
                    ci = np.zeros(0, np.int64)
                else:
                    ri, ci = aca(lambda i: kernels.block(kernel_id, kparams, pts, R[i:i + 1], F)[0],
                                 lambda j: kernels.block(kernel_id, kparams, pts, R, F[j:j + 1])[:, 0],
                                 R.size, F.size, eps)
                sk, fp = R[ri], F[ci]
                self.sk[l][B], self.fp[l][B] = sk, fp
                k = sk.size
                if k == 0:
                    self.U[l][B] = np.zeros((R.size, 0))
                    continue
                # V^* = A(fp, sk)^{-1} A(fp, R); U = V for u = v, symmetric K (R10)
                Afs = kernels.block(kernel_id, kparams, pts, fp, sk)
                AfR = kernels.block(kernel_id, kparams, pts, fp, R)
                X = np.linalg.solve(Afs, AfR)
                self.U[l][B] = np.ascontiguousarray(X.T)

    def rank(self, l, B):
        return self.sk[l][B].size

    def child_rows(self, l, P):
        """Row offsets of each child's block inside U[l][P] (children in Morton order)."""
        out, o = {}, 0
        for c in self.t.children(l, P):
            kc = self.sk[l + 1][c].size
            out[c] = (o, o + kc)
            o += kc
        return out
