"""Pins for oracle/nnca.py and oracle/linalg.py (closed forms, exact identities, dense blocks)."""
import numpy as np
import pytest

from oracle import dense, kernels
from oracle.factor import AIFMM
from oracle.linalg import pick, pivoted_qr_extend
from oracle.nnca import aca
from paper_2301_12704_b200 import workloads as W


def test_kernel_closed_forms():
    X = np.array([[0.0, 0.0], [3.0, 4.0]])
    A = kernels.entries(0, (10.0, 0.0), X, X, [0, 1], [0, 1])
    assert A[0, 0] == 10.0 and np.isclose(A[0, 1], np.log(5.0))
    A = kernels.entries(1, (1.01, 0.1), X, X, [0, 1], [0, 1])
    assert A[1, 1] == 1.01 and np.isclose(A[0, 1], np.exp(-50.0))
    A = kernels.entries(2, (128.0, 0.0), X, X, [0, 1], [0, 1])
    assert np.isclose(A[1, 0], 0.2)
    with pytest.raises(FloatingPointError):
        kernels.entries(2, (1.0, 0.0), X[[0, 0]], X[[0, 0]], [0, 1], [0, 1])


def test_pick_tie_window():
    assert pick(np.array([1.0, 3.0, 3.0 * (1 - 1e-12), -3.0])) == 1
    assert pick(np.array([0.0, 0.0])) is None
    assert pick(np.array([5.0, 1.0]), np.array([True, False])) == 1


def test_aca_exact_low_rank():
    rng = np.random.default_rng(0)
    for r in (1, 3, 7):
        M = rng.standard_normal((40, r)) @ rng.standard_normal((r, 55))
        rp, cp = aca(lambda i: M[i], lambda j: M[:, j], 40, 55, 1e-12)
        assert len(rp) == r                       # stops at the exact rank
        # skeleton reconstruction M = M[:, cp] M[rp, cp]^{-1} M[rp, :]
        R = M[:, cp] @ np.linalg.solve(M[np.ix_(rp, cp)], M[rp, :])
        assert np.linalg.norm(R - M) <= 1e-10 * np.linalg.norm(M)


def test_pivoted_qr_truncation_contract():
    rng = np.random.default_rng(1)
    for r in (0, 2, 9):
        F = rng.standard_normal((30, r)) @ rng.standard_normal((r, 70)) if r else np.zeros((30, 70))
        if r:
            F = F + 1e-9 * rng.standard_normal(F.shape)
        tau = 1e-6 * max(np.linalg.norm(F), 1e-300)
        Q, t = pivoted_qr_extend(F, np.zeros((30, 0)), tau, 0, 30)
        assert t == r == Q.shape[1]
        if r:
            assert np.abs(Q.T @ Q - np.eye(r)).max() < 1e-12
        assert np.linalg.norm(F - Q @ (Q.T @ F)) <= tau


@pytest.mark.parametrize("kid,kp,kind", [(0, (10.0, 0.0), "grid"), (1, (1.01, 0.1), "uniform_pm1"),
                                         (2, (100.0, 0.0), "uniform_pm1")])
@pytest.mark.parametrize("tol", [1e-6, 1e-10])
def test_nnca_far_blocks_within_10tol(kid, kp, kind, tol):
    """BASELINE oracle self-check: every NNCA far block at every level has relative
    Frobenius error <= 10 * tol against the dense block (N <= 2048)."""
    n = 1024 if kind == "grid" else 2048
    pts = W.make_points(kind, n, 2, 3)
    o = AIFMM(pts, kid, kp, 16, tol)
    errs = dense.far_block_errors(o)
    assert len(errs) > 100
    assert max(e[3] for e in errs) <= 10 * tol


def test_nnca_interpolative_identity_and_rank_monotone():
    pts, _ = W.small_problem(d=2, n=2048, seed=4)
    ranks = []
    for tol in (1e-4, 1e-7, 1e-10):
        o = AIFMM(pts, 0, (10.0, 0.0), 32, tol)
        nn = o.nnca
        tot = 0
        for l in nn.U:
            for B, U in nn.U[l].items():
                R, sk = nn.R[l][B], nn.sk[l][B]
                pos = [int(np.flatnonzero(R == s)[0]) for s in sk]
                # U_B restricted to the skeleton rows is the identity
                if sk.size:
                    # exact up to cond(A(fp, sk)) * eps (LU solve rounding)
                    kap = np.linalg.cond(kernels.block(0, (10.0, 0.0), o.tree.points, nn.fp[l][B], sk))
                    assert np.abs(U[pos] - np.eye(sk.size)).max() <= 100 * kap * 2.2e-16
                tot += sk.size
        ranks.append(tot)
    assert ranks[0] <= ranks[1] <= ranks[2]
