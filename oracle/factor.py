"""AIFMM factorization and solve (oracle; test infrastructure only).

Follows PAPER.md §3 step by step:
  * extended sparse system (§3.1): per box i at level l the variables
    x_i (particles; at l < L the stacked child multipoles, Eq. P:414-416), z_i (locals),
    y_i (multipoles); rows X_i (Eq. EquationX), Y_i (Eq. EquationY, -I on y_i
    per the legend P:578) and Z_i (Eq. EqXl: U_i^dag z_P + sum_IL A_ic y_c - z_i = 0,
    which is the row block of X_P at level l-1; z^(1) = 0);
  * elimination of (x_i, z_i) with rows (X_i, Y_i), fill-ins per Table 4 /
    the four cases, Eq. X2;
  * Algorithm 3: far fill-ins are accumulated and compressed/redirected once,
    just before one of their members is eliminated -- colour-batched (R12);
  * P2P / P2L / M2P compression and redirection (§3.2.1-3.2.3);
  * top dense solve of the level-2 multipoles (Alg. 4 line 1 P:1173);
  * Algorithm 4 back substitution, factor independent of b (Remark P:1186-1188).

Block storage (per level): near[(p,q)] is the coupling between the LIVE row of p (X_p if p
is not eliminated, else Z_p) and the LIVE column of q (x_q, else y_q), q in N(p);
A[(p,q)] is the (Z_p, y_q) M2L block for q in IL(p); F[(p,q)] is the pending far fill-in
(P2P / P2L / M2P by elimination state, Table) for IL pairs at Chebyshev distance 2.

Readings used here: R12 colour-batched Alg. 3; R13 orthonormalise U, V at the
start of each level by an exact change of variables (the update derivations assume
U~^* U~ = I); R14 project-then-compress RRQR with truncation
tol_c * ||F||_F and Galerkin redirection A <- U~^*(U A V^* + F) V~, which with orthonormal
bases equals L A R^* + R~^* and zero-pads the other
M2L, M2M, L2L blocks; R15 + R27 equal box ranks |z_i| = |y_i| (needed for a
square pivot [[K, U],[V^*, 0]]): one-sided compression, V's new columns = U's, capped at m_i;
R16 pivot inverse G = P_i^{-1} by LU with partial pivoting; R17 (Z_i, y_i) = -G22;
R8b the RRQR runs on the triangular factor of the projected candidate matrix (tri_root).
"""
from __future__ import annotations

import numpy as np

from . import kernels
from .tree import Tree, build_lists, greedy_colours, chebyshev
from .nnca import NNCA
from .linalg import pivoted_qr_extend


def _pad(M, r, c):
    out = np.zeros((r, c))
    out[:M.shape[0], :M.shape[1]] = M
    return out


def tri_root(W):
    """R8b two-stage RRQR: W^T = Q R (Householder), return R^T (m x min(m, n)).

    For every projector P acting on the left, ||(I - P) R^T||_F = ||(I - P) W||_F and
    range(R^T) = range(W), so the truncated pivoted QR of R^T is a rank-revealing QR of W
    with exactly the truncation criterion of R8 -- on an m x m instead of an m x n matrix."""
    if W.shape[1] == 0:
        return W
    R = np.linalg.qr(W.T, mode="r")
    return np.ascontiguousarray(R.T)


class Level:
    pass


class AIFMM:
    """Oracle AIFMM: build (tree, lists, colours, NNCA), factor, solve."""

    def __init__(self, points, kernel_id, kparams, leaf_size, tol, tol_c=None, nnca_eps=None, algorithm=3):
        self.kid, self.kp = kernel_id, tuple(kparams)
        # algorithm = 3: Alg. 3, far fill-ins compressed once, just before one of
        # their members is eliminated; algorithm = 2: Alg. 2, compressed as soon as
        # they are created or updated -- here right after the colour that created them (SURVEY
        # §8(f) row f2, reading R29)
        if algorithm not in (2, 3):
            raise ValueError("algorithm must be 2 or 3")
        self.algorithm = algorithm
        self.tol = tol
        self.tol_c = tol if tol_c is None else tol_c
        self.tree = Tree(points, leaf_size)
        self.near, self.il = build_lists(self.tree)
        self.colour = {l: greedy_colours(self.tree, self.near[l]) for l in self.near}
        # R18: eps_ACA = tol / 100 meets the 10*tol per-block bound on all three kernels
        self.nnca = NNCA(self.tree, self.near, self.il, kernel_id, self.kp,
                         tol / 100.0 if nnca_eps is None else nnca_eps)
        self.levels = {}
        self.stats = {"compressions": 0, "rank_growth": {}, "max_rank": {}}
        self.factored = False

    # ------------------------------------------------------------------ helpers
    def _dist2_far(self, l, p, q):
        return q in self.il[l][p] and chebyshev(self.tree, l, p, q) == 2

    def _live(self, lv, b):
        return lv.k[b] if lv.E[b] else lv.m[b]

    # ------------------------------------------------------------------ level setup
    def _setup_level(self, l, prev):
        t, nn = self.tree, self.nnca
        lv = Level()
        lv.l = l
        lv.boxes = sorted(self.near[l])
        lv.m, lv.k, lv.U, lv.V, lv.Ud, lv.Vd = {}, {}, {}, {}, {}, {}
        lv.near, lv.A, lv.F = {}, {}, {}
        lv.E = {b: False for b in lv.boxes}
        lv.pending = set()
        lv.rec = {}
        lv.xoff = {}
        for b in lv.boxes:
            if l == t.L:
                lv.m[b] = t.count(l, b)
                lv.U[b] = nn.U[l][b].copy()
            else:
                ch = t.children(l, b)
                o = 0
                for c in ch:
                    lv.xoff[(b, c)] = (o, o + prev.k[c])
                    o += prev.k[c]
                lv.m[b] = o
                lv.U[b] = np.concatenate([prev.Ud[c] for c in ch], axis=0) if ch else np.zeros((0, nn.rank(l, b)))
            lv.V[b] = lv.U[b].copy() if l == t.L else (
                np.concatenate([prev.Vd[c] for c in t.children(l, b)], axis=0) if t.children(l, b) else np.zeros((0, nn.rank(l, b))))
            lv.k[b] = nn.rank(l, b)
            if l > 2:
                P = b >> t.d
                r0, r1 = nn.child_rows(l - 1, P)[b]
                lv.Ud[b] = nn.U[l - 1][P][r0:r1].copy()       # L2L U_b^dag
                lv.Vd[b] = lv.Ud[b].copy()                     # M2M V_b^dag, = U^dag (R10)
            else:
                lv.Ud[b] = np.zeros((lv.k[b], 0))
                lv.Vd[b] = np.zeros((lv.k[b], 0))
        # near blocks K^(l)
        for p in lv.boxes:
            for q in self.near[l][p]:
                if l == t.L:
                    a0, a1 = t.point_range(l, p)
                    b0, b1 = t.point_range(l, q)
                    lv.near[(p, q)] = kernels.block(self.kid, self.kp, t.points,
                                                     np.arange(a0, a1), np.arange(b0, b1))
                else:
                    M = np.zeros((lv.m[p], lv.m[q]))
                    for c in t.children(l, p):
                        r0, r1 = lv.xoff[(p, c)]
                        for c2 in t.children(l, q):
                            s0, s1 = lv.xoff[(q, c2)]
                            blk = prev.near[(c, c2)] if c2 in self.near[l + 1][c] else prev.A[(c, c2)]
                            M[r0:r1, s0:s1] = blk
                    lv.near[(p, q)] = M
            # M2L A_pq = A(sk p, sk q)
            for q in self.il[l][p]:
                lv.A[(p, q)] = kernels.block(self.kid, self.kp, t.points, nn.sk[l][p], nn.sk[l][q])
        self._orthonormalise(lv)
        return lv

    def _orthonormalise(self, lv):
        """R13: U_b = Q T, z~_b = T z_b: U_b <- Q, rows of Z_b (U_b^dag, A_bc) <- T (.);
        V_b = Q' T', y_b = T'^T y~_b: columns of y_b (A_db, V_b^dag*) <- (.) T'^T."""
        l = lv.l
        for b in lv.boxes:
            if lv.k[b] == 0:
                continue
            Q, T = np.linalg.qr(lv.U[b])
            lv.U[b] = Q
            lv.Ud[b] = T @ lv.Ud[b]
            for c in self.il[l][b]:
                lv.A[(b, c)] = T @ lv.A[(b, c)]
            Q2, T2 = np.linalg.qr(lv.V[b])
            lv.V[b] = Q2
            lv.Vd[b] = T2 @ lv.Vd[b]
            for d in self.il[l][b]:
                lv.A[(d, b)] = lv.A[(d, b)] @ T2.T

    # ------------------------------------------------------------------ Alg. 3 compression
    def _compress(self, lv, S):
        """Compress and redirect every pending far pair in S (Alg. 3 lines P:1118-1129)."""
        l = lv.l
        part = {}
        for (a, b) in S:
            part.setdefault(a, []).append(b)
            part.setdefault(b, []).append(a)
        affected = sorted(b for b in part if not lv.E[b])
        newU = {}
        for b in affected:
            ps = sorted(part[b])
            m, k = lv.m[b], lv.k[b]
            # reading R27: every kernel here is symmetric (A_ij = A_ji, targets = sources),
            # so the column-side fill-ins are the transposes of the row-side ones (F_pb^T = F_bp)
            # and the V-side basis extension of P:852-863 equals the U-side one in exact
            # arithmetic: it is computed once, from row X_b, and V_b's new columns are U_b's (the
            # pivots stay [[K, U], [U^T, 0]], square: |z_b| = |y_b| as P:753 needs, R15)
            FU = np.concatenate([lv.F[(b, q)] for q in ps], axis=1)       # row X_b
            nU = np.linalg.norm(FU)
            WU = tri_root(FU - lv.U[b] @ (lv.U[b].T @ FU))
            # R8 with tmin = 0: the columns taken are exactly the t_trunc of the truncation test
            QU, tt = pivoted_qr_extend(WU, lv.U[b], self.tol_c * nU, 0, m - k)
            assert QU.shape[1] == tt
            newU[b] = np.concatenate([lv.U[b], QU], axis=1)
            self.stats["compressions"] += 1
            g = self.stats["rank_growth"].setdefault(l, 0)
            self.stats["rank_growth"][l] = g + tt
        # zero-pad Z_b rows / y_b columns (other M2L, M2M, L2L updates)
        for b in affected:
            k1 = newU[b].shape[1]
            if k1 == lv.k[b]:
                continue
            lv.Ud[b] = _pad(lv.Ud[b], k1, lv.Ud[b].shape[1])
            lv.Vd[b] = _pad(lv.Vd[b], k1, lv.Vd[b].shape[1])
            for c in self.il[l][b]:
                A = lv.A[(b, c)]
                lv.A[(b, c)] = _pad(A, k1, A.shape[1])
                A = lv.A[(c, b)]
                lv.A[(c, b)] = _pad(A, A.shape[0], k1)
            lv.k[b] = k1
        for b in affected:
            lv.U[b], lv.V[b] = newU[b], newU[b].copy()
        # redirect the fill-ins (Galerkin projection onto the new bases)
        for (a, b) in S:
            for (x, y) in ((a, b), (b, a)):
                Fxy = lv.F.pop((x, y))
                if not lv.E[x] and not lv.E[y]:       # P2P
                    lv.A[(x, y)] += lv.U[x].T @ Fxy @ lv.V[y]
                elif lv.E[x] and not lv.E[y]:         # P2L
                    lv.A[(x, y)] += Fxy @ lv.V[y]
                elif not lv.E[x] and lv.E[y]:         # M2P
                    lv.A[(x, y)] += lv.U[x].T @ Fxy
                else:
                    raise AssertionError("both eliminated: never pending (A17)")
            lv.pending.discard((a, b))

    # ------------------------------------------------------------------ elimination
    def _target(self, lv, p, q):
        l = lv.l
        if q in self.near[l][p]:
            return ("near", (p, q))
        if lv.E[p] and lv.E[q]:
            return ("A", (p, q))
        assert self._dist2_far(l, p, q)
        if (p, q) not in lv.F:
            lv.F[(p, q)] = np.zeros((self._live(lv, p), self._live(lv, q)))
        lv.pending.add((min(p, q), max(p, q)))
        return ("F", (p, q))

    def _eliminate(self, lv, i, skip_schur=False):
        l = lv.l
        m, k = lv.m[i], lv.k[i]
        P = np.zeros((m + k, m + k))
        P[:m, :m] = lv.near[(i, i)]
        P[:m, m:] = lv.U[i]
        P[m:, :m] = lv.V[i].T
        G = np.linalg.inv(P) if m + k > 0 else np.zeros((0, 0))
        nb = [q for q in self.near[l][i] if q != i]
        R = {q: (lv.near[(i, q)], bool(lv.E[q])) for q in nb}      # row X_i
        C = {p: (lv.near[(p, i)], bool(lv.E[p])) for p in nb}      # column x_i
        lv.rec[i] = {"G": G, "m": m, "k": k, "R": R, "C": C}
        W = {q: G[:, :m] @ R[q][0] for q in nb}
        # R28: with k = m the orthonormal U_i (R13) is square, P_i^{-1} = [[0, U], [U^T, -U^T K U]]
        # (V = U, R27): G11 = 0 exactly, so the box makes no Schur update and no fill-in.  Decided
        # when the box's colour begins (a box the colour's compression fills up keeps its terms,
        # which are then zero up to rounding).
        if not skip_schur:
            for p in nb:
                Cp = C[p][0]
                for q in nb:
                    kind, key = self._target(lv, p, q)
                    store = {"near": lv.near, "A": lv.A, "F": lv.F}[kind]
                    store[key] = store[key] - Cp @ W[q][:m]
        for p in nb:
            lv.near[(p, i)] = C[p][0] @ G[:m, m:]           # (X_p|Z_p, y_i) += C G12
        for q in nb:
            lv.near[(i, q)] = W[q][m:]                       # (Z_i, x_q|y_q) += G21 R
        lv.near[(i, i)] = -G[m:, m:]                         # (Z_i, y_i) = -G22 (R17)

    def factor(self):
        t = self.tree
        prev = None
        for l in range(t.L, 1, -1):
            lv = self._setup_level(l, prev)
            ncol = max(self.colour[l].values()) + 1
            for c in range(ncol):
                cset = {b for b in lv.boxes if self.colour[l][b] == c}
                S = sorted(p for p in lv.pending if p[0] in cset or p[1] in cset)
                # R28 is decided when the colour begins (before its compression)
                full = {i for i in cset if lv.m[i] > 0 and lv.k[i] >= lv.m[i]}
                if S:
                    self._compress(lv, S)
                for i in sorted(cset):
                    self._eliminate(lv, i, skip_schur=i in full)
                for i in cset:
                    lv.E[i] = True
                if self.algorithm == 2 and lv.pending:       # Alg. 2: compress on creation
                    self._compress(lv, sorted(lv.pending))
            assert not lv.pending and not lv.F, "pending far fill-ins at level end"
            self.stats["max_rank"][l] = max(lv.k.values())
            self.levels[l] = lv
            prev = lv
        # top: (Z_p, y_q) over level-2 boxes
        lv = self.levels[2]
        offs, o = {}, 0
        for b in lv.boxes:
            offs[b] = (o, o + lv.k[b])
            o += lv.k[b]
        M = np.zeros((o, o))
        for p in lv.boxes:
            for q in lv.boxes:
                blk = lv.near[(p, q)] if q in self.near[2][p] else lv.A[(p, q)]
                M[offs[p][0]:offs[p][1], offs[q][0]:offs[q][1]] = blk
        self.top = M
        self.top_offs = offs
        self.factored = True
        return self

    # ------------------------------------------------------------------ Alg. 4 solve
    def solve(self, B):
        assert self.factored
        t = self.tree
        B = np.asarray(B, dtype=np.float64)
        one = B.ndim == 1
        if one:
            B = B[:, None]
        nr = B.shape[1]
        Bs = B[t.perm]
        bX, bZ = {}, {}
        for l in range(t.L, 1, -1):
            lv = self.levels[l]
            bX[l], bZ[l] = {}, {}
            for b in lv.boxes:
                if l == t.L:
                    a0, a1 = t.point_range(l, b)
                    bX[l][b] = Bs[a0:a1].copy()
                else:
                    ch = t.children(l, b)
                    bX[l][b] = (np.concatenate([bZ[l + 1][c] for c in ch], axis=0)
                                if ch else np.zeros((0, nr)))
                bZ[l][b] = np.zeros((lv.k[b], nr))
            ncol = max(self.colour[l].values()) + 1
            for c in range(ncol):
                for i in sorted(b for b in lv.boxes if self.colour[l][b] == c):
                    r = lv.rec[i]
                    m = r["m"]
                    w = r["G"][:, :m] @ bX[l][i]
                    for p, (Cb, pz) in r["C"].items():
                        if pz:
                            bZ[l][p] -= Cb @ w[:m]
                        else:
                            bX[l][p] -= Cb @ w[:m]
                    bZ[l][i] += w[m:]
        lv2 = self.levels[2]
        rhs = np.concatenate([bZ[2][b] for b in lv2.boxes], axis=0)
        ytop = np.linalg.solve(self.top, rhs) if rhs.shape[0] else rhs
        y = {2: {b: ytop[self.top_offs[b][0]:self.top_offs[b][1]] for b in lv2.boxes}}
        x = {}
        for l in range(2, t.L + 1):
            lv = self.levels[l]
            x[l] = {}
            ncol = max(self.colour[l].values()) + 1
            for c in range(ncol - 1, -1, -1):
                for i in sorted((b for b in lv.boxes if self.colour[l][b] == c), reverse=True):
                    r = lv.rec[i]
                    m = r["m"]
                    rhs = bX[l][i].copy()
                    for q, (Rb, qy) in r["R"].items():
                        rhs -= Rb @ (y[l][q] if qy else x[l][q])
                    xz = r["G"] @ np.concatenate([rhs, y[l][i]], axis=0)
                    x[l][i] = xz[:m]
            if l < t.L:
                y[l + 1] = {}
                for b in lv.boxes:
                    for c in t.children(l, b):
                        r0, r1 = lv.xoff[(b, c)]
                        y[l + 1][c] = x[l][b][r0:r1]
        xs = np.zeros((t.n, nr))
        for b in self.levels[t.L].boxes:
            a0, a1 = t.point_range(t.L, b)
            xs[a0:a1] = x[t.L][b]
        X = np.zeros_like(xs)
        X[t.perm] = xs
        return X[:, 0] if one else X
