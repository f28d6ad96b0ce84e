"""H2 matrix-vector product with the NNCA operators, and restarted GMRES (oracle; test
infrastructure only -- only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
may import it).

SURVEY §8(a) row a8 / BASELINE config 5: AIFMM at a loose tolerance is the preconditioner of
GMRES(30) whose matrix-vector products use an NNCA (H2) approximation of A at a tight
tolerance (§5 Exp. 5: "AIFMM as a preconditioner", iterative solves with
the FMM matvec).

H2 product (Eq. NCA P:347-357 with the nested operators of P:360-367, Table), per
level l = L..2 on the tree of the oracle:
  upward   q_B = V_B^* x_B             (P2M at the leaf, V_B = U_B by R10)
           q_B = V_B^* [q_c]_c          (M2M: the particles of B are its children's multipoles,
                                          Eq. P:414-416)
  M2L      l_B = sum_{D in IL(B)} A(sk_B, sk_D) q_D      (A_BD = A_{t^{B,i} s^{D,o}})
  downward l_c += U_P[rows of c] l_P    (L2L, U_B^dag of P:364)
  leaf     y_B = sum_{X in N(B)} K_BX x_X + U_B l_B      (near field P:366 + L2P)
This is the product with the densified matrix of dense.h2_matrix, written as the fast
algorithm; it is pinned against that densification and against the exact A.

GMRES (right preconditioned, restart m, modified Gram-Schmidt Arnoldi, Givens rotations):
solve (A M^{-1}) u = b, x = M^{-1} u, stopping when the Arnoldi residual estimate
|g_{j+1}| <= rtol ||b||; the true residual ||b - A x|| is recomputed at each restart
(Saad, Iterative Methods for Sparse Linear Systems, Alg. 9.5 / 6.11).
"""
from __future__ import annotations

import numpy as np

from . import kernels
from .nnca import NNCA
from .tree import Tree, build_lists


class H2:
    """NNCA-compressed representation of A at tolerance tol (eps_ACA = tol/100, reading R18)."""

    def __init__(self, points, kernel_id, kparams, leaf_size, tol, tree=None, near=None, il=None):
        self.kid, self.kp = kernel_id, tuple(kparams)
        self.tree = Tree(points, leaf_size) if tree is None else tree
        if near is None:
            near, il = build_lists(self.tree)
        self.near, self.il = near, il
        self.nnca = NNCA(self.tree, near, il, kernel_id, self.kp, tol / 100.0)

    def matvec(self, x):
        """y = A_H2 x (user order; x of shape (N,) or (N, r))."""
        t, nn = self.tree, self.nnca
        X = np.asarray(x, dtype=np.float64)
        one = X.ndim == 1
        if one:
            X = X[:, None]
        xs = X[t.perm]
        L = t.L
        pts = t.points
        q = {}
        for l in range(L, 1, -1):                         # upward (P2M, M2M)
            q[l] = {}
            for B in sorted(self.near[l]):
                if l == L:
                    a, b = t.point_range(l, B)
                    src = xs[a:b]
                else:
                    parts = [q[l + 1][c] for c in t.children(l, B)]
                    src = np.concatenate(parts, axis=0) if parts else np.zeros((0, X.shape[1]))
                q[l][B] = nn.U[l][B].T @ src
        loc = {}
        for l in range(2, L + 1):                         # M2L
            loc[l] = {}
            for B in sorted(self.near[l]):
                acc = np.zeros((nn.rank(l, B), X.shape[1]))
                for D in self.il[l][B]:
                    acc += kernels.block(self.kid, self.kp, pts, nn.sk[l][B], nn.sk[l][D]) @ q[l][D]
                loc[l][B] = acc
        for l in range(2, L):                             # downward (L2L)
            for P in sorted(self.near[l]):
                rows = nn.child_rows(l, P)
                for c, (r0, r1) in rows.items():
                    loc[l + 1][c] = loc[l + 1][c] + nn.U[l][P][r0:r1] @ loc[l][P]
        ys = np.zeros_like(xs)
        for B in sorted(self.near[L]):                    # near field + L2P
            a, b = t.point_range(L, B)
            acc = nn.U[L][B] @ loc[L][B]
            for Xb in self.near[L][B]:
                c0, c1 = t.point_range(L, Xb)
                acc = acc + kernels.block(self.kid, self.kp, pts, np.arange(a, b), np.arange(c0, c1)) @ xs[c0:c1]
            ys[a:b] = acc
        Y = np.zeros_like(ys)
        Y[t.perm] = ys
        return Y[:, 0] if one else Y


def gmres(matvec, b, precond=None, restart=30, rtol=1e-10, maxit=1000):
    """Right-preconditioned restarted GMRES (MGS Arnoldi, Givens rotations).

    Returns (x, iterations, relative residual ||b - A x|| / ||b|| by `matvec`)."""
    b = np.asarray(b, dtype=np.float64)
    n = b.shape[0]
    M = precond if precond is not None else (lambda v: v)
    x = np.zeros(n)
    bnorm = np.linalg.norm(b)
    if bnorm == 0.0:
        return x, 0, 0.0
    it = 0
    r = b - matvec(x)
    beta = np.linalg.norm(r)
    while it < maxit and beta > rtol * bnorm:
        V = np.zeros((restart + 1, n))
        H = np.zeros((restart + 1, restart))
        cs, sn = np.zeros(restart), np.zeros(restart)
        g = np.zeros(restart + 1)
        g[0] = beta
        V[0] = r / beta
        j = 0
        while j < restart and it < maxit:
            w = matvec(M(V[j]))
            for i in range(j + 1):                        # modified Gram-Schmidt
                H[i, j] = w @ V[i]
                w = w - H[i, j] * V[i]
            H[j + 1, j] = np.linalg.norm(w)
            if H[j + 1, j] != 0.0:
                V[j + 1] = w / H[j + 1, j]
            for i in range(j):                            # previous rotations
                h0, h1 = H[i, j], H[i + 1, j]
                H[i, j] = cs[i] * h0 + sn[i] * h1
                H[i + 1, j] = -sn[i] * h0 + cs[i] * h1
            den = np.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = (1.0, 0.0) if den == 0.0 else (H[j, j] / den, H[j + 1, j] / den)
            H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            j += 1
            it += 1
            if abs(g[j]) <= rtol * bnorm:
                break
        y = np.zeros(j)                                   # back substitution H[:j,:j] y = g[:j]
        for i in range(j - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:j] @ y[i + 1:j]) / H[i, i]
        x = x + M(V[:j].T @ y)
        r = b - matvec(x)
        beta = np.linalg.norm(r)
    return x, it, float(beta / bnorm)


def block_diagonal_precond(tree, kernel_id, kparams):
    """The block-diagonal preconditioner of the paper's comparison (I_BD, table
    P:1684-1700): M = blockdiag(A(points(b), points(b))) over the leaves b
    of the tree, each block written out exactly (kernels.block) and inverted (numpy.linalg.inv).
    Returns v -> M^{-1} v in user order."""
    L = tree.L
    blocks = []
    for b in tree.nonempty(L):
        a0, a1 = tree.point_range(L, b)
        idx = np.arange(a0, a1)
        blocks.append((a0, a1, np.linalg.inv(kernels.block(kernel_id, kparams, tree.points, idx, idx))))

    def apply(v):
        vs = np.asarray(v, dtype=np.float64)[tree.perm]
        out = np.empty_like(vs)
        for a0, a1, Binv in blocks:
            out[a0:a1] = Binv @ vs[a0:a1]
        res = np.empty_like(out)
        res[tree.perm] = out
        return res
    return apply
