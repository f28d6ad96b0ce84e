"""Pins for oracle/h2.py: the NNCA (H2) matrix-vector product and restarted GMRES
(BASELINE config 5).  Pinned against the densified NNCA matrix, the exact
kernel matrix, linearity, and closed-form Krylov behaviour."""
import numpy as np
import pytest

from oracle import dense
from oracle.factor import AIFMM
from oracle.h2 import H2, gmres
from paper_2301_12704_b200 import workloads as W


@pytest.mark.parametrize("d,kind,kid,kp", [(2, "uniform_pm1", 0, (10.0, 0.0)), (3, "uniform_01", 2, (100.0, 0.0))])
def test_h2_matvec_equals_densified_nnca_and_approximates_A(d, kind, kid, kp):
    n, tol = 1500, 1e-8
    pts = W.make_points(kind, n, d, 8)
    o = AIFMM(pts, kid, kp, 24, tol)
    h = H2(pts, kid, kp, 24, tol, tree=o.tree, near=o.near, il=o.il)
    x = W.make_rhs(n, 2, 8)
    y = h.matvec(x)
    # the fast algorithm is the product with the densified NNCA matrix (same operators)
    yd = dense.h2_matrix(o) @ x
    assert np.linalg.norm(y - yd) <= 1e-12 * np.linalg.norm(yd)
    # and approximates the exact kernel matrix at the NNCA accuracy (<= 10 tol per block)
    A = dense.dense_matrix(pts, kid, kp)
    assert np.linalg.norm(y - A @ x) <= 10 * tol * np.linalg.norm(A) * np.linalg.norm(x)
    # linearity
    a, b = 0.7, -1.3
    assert np.allclose(h.matvec(a * x[:, 0] + b * x[:, 1]), a * y[:, 0] + b * y[:, 1], rtol=0, atol=1e-12 * np.abs(y).max())


def test_gmres_dense_and_closed_forms():
    rng = np.random.default_rng(2)
    n = 60
    A = rng.standard_normal((n, n)) + 12 * np.eye(n)
    b = rng.standard_normal(n)
    x, it, rr = gmres(lambda v: A @ v, b, restart=30, rtol=1e-12)
    xe = np.linalg.solve(A, b)
    assert rr <= 1e-12 and np.linalg.norm(x - xe) <= 1e-10 * np.linalg.norm(xe)
    # exact preconditioner: one iteration
    Ai = np.linalg.inv(A)
    x, it, rr = gmres(lambda v: A @ v, b, precond=lambda v: Ai @ v, rtol=1e-10)
    assert it == 1 and rr <= 1e-10
    # a diagonal matrix with 5 distinct eigenvalues: the Krylov space is exhausted after 5 steps
    D = np.repeat([1.0, 2.0, 3.0, 5.0, 8.0], 12)
    x, it, rr = gmres(lambda v: D * v, b, rtol=1e-12)
    assert it <= 5 and rr <= 1e-12
    # restarts: a small restart length still converges, with more iterations
    x2, it2, rr2 = gmres(lambda v: A @ v, b, restart=3, rtol=1e-12, maxit=2000)
    assert rr2 <= 1e-12 and it2 >= 3


def test_aifmm_preconditioned_gmres_config5_style():
    """Config 5 in miniature: 3D uniform points in the unit cube, 1/r with A_ii = 100, NNCA
    matvec at 1e-10, AIFMM factor at the loose tolerance 1e-3 as right preconditioner,
    GMRES(30) to 1e-10 -- fewer iterations than unpreconditioned GMRES, and the exact residual
    is at the matvec accuracy."""
    n = 1200
    pts = W.make_points("uniform_01", n, 3, 4)
    b = W.make_rhs(n, 1, 4)[:, 0]
    kp = (100.0, 0.0)
    h = H2(pts, 2, kp, 32, 1e-10)
    P = AIFMM(pts, 2, kp, 32, 1e-3).factor()
    x, it, rr = gmres(h.matvec, b, precond=P.solve, restart=30, rtol=1e-10)
    assert rr <= 1e-10
    # unpreconditioned GMRES has not converged after the same number of iterations
    _, it0, rr0 = gmres(h.matvec, b, restart=30, rtol=1e-10, maxit=it)
    assert rr0 > 1e-10
    A = dense.dense_matrix(pts, 2, kp)
    assert np.linalg.norm(A @ x - b) <= 1e-8 * np.linalg.norm(b)


def test_block_diagonal_precond_inverts_leaf_blocks():
    """oracle/h2.py: block_diagonal_precond applied to blockdiag(A) x gives x back (the dense
    block-diagonal part written out from the exact matrix, same leaves), in user order."""
    from oracle.h2 import block_diagonal_precond
    from oracle.tree import Tree
    pts, _ = W.small_problem(d=2, n=700, seed=3)
    kp = (10.0, 0.0)
    t = Tree(pts, 30)
    leaf_of = np.empty(700, dtype=np.int64)
    for b in t.nonempty(t.L):
        a0, a1 = t.point_range(t.L, b)
        leaf_of[t.perm[a0:a1]] = b
    A = dense.dense_matrix(pts, 0, kp)
    Abd = np.where(leaf_of[:, None] == leaf_of[None, :], A, 0.0)
    x = np.random.default_rng(0).standard_normal(700)
    M = block_diagonal_precond(t, 0, kp)
    assert np.linalg.norm(M(Abd @ x) - x) <= 1e-10 * np.linalg.norm(x)
