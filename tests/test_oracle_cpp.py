"""Pins for the serial C++ oracle (oracle/cpp/aifmm_oracle.cpp via oracle/cpp.py).

The same pins as the numpy oracle (test_oracle_factor.py: dense LU at tol 1e-14, exact
algebra with tol_c = 0, residual monotone in tol, b = 0, multi-RHS, the paper's Exp. 3 row)
plus agreement with the numpy oracle (integer outputs bit-exact; solutions to rounding level)
and bit-identical results for every OpenMP thread count."""
import numpy as np
import pytest

from oracle import dense
from oracle.cpp import CppAIFMM, OracleError
from oracle.factor import AIFMM
from paper_2301_12704_b200 import workloads as W


def _paper_exp3(n):
    return (2, (float(np.sqrt(1000.0 * n)), 0.0))


CASES = [
    ("grid2d_log", "grid", 4096, 2, 0, (10.0, 0.0), 64, 1e-8),
    ("rand2d_log_ragged", "uniform_pm1", 3000, 2, 0, (10.0, 0.0), 40, 1e-8),
    ("rand2d_matern", "uniform_pm1", 2500, 2, 1, (1.01, 0.1), 32, 1e-6),
    ("rand3d_invr", "uniform_01", 3000, 3, 2, (100.0, 0.0), 32, 1e-7),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_cpp_matches_numpy_oracle(case):
    """Integer outputs (tree permutation, offsets, N/IL lists, colours, NNCA ranks and
    skeletons) bit-exact with the numpy oracle; solutions equal to rounding level."""
    name, kind, n, d, kid, kp, leaf, tol = case
    pts = W.make_points(kind, n, d, 21)
    b = W.make_rhs(n, 2, 21)
    o = AIFMM(pts, kid, kp, leaf, tol).factor()
    c = CppAIFMM(pts, kid, kp, leaf, tol).factor()
    assert c.L == o.tree.L
    assert np.array_equal(c.perm(), o.tree.perm)
    for l in range(0, c.L + 1):
        assert np.array_equal(c.offsets(l), o.tree.off[l])
    for l in range(2, c.L + 1):
        nptr, nidx, iptr, iidx = c.lists(l)
        col = c.colours(l)
        rk = c.ranks(l, 0)
        for bx in range(1 << (d * l)):
            if bx in o.near[l]:
                assert list(nidx[nptr[bx]:nptr[bx + 1]]) == o.near[l][bx]
                assert list(iidx[iptr[bx]:iptr[bx + 1]]) == o.il[l][bx]
                assert col[bx] == o.colour[l][bx]
                assert rk[bx] == o.nnca.rank(l, bx)
                assert np.array_equal(c.skeleton(l, bx), o.nnca.sk[l][bx])
            else:
                assert nptr[bx + 1] == nptr[bx] and col[bx] == -1
    x, xo = c.solve(b), o.solve(b)
    assert np.linalg.norm(x - xo) / np.linalg.norm(xo) <= 10 * tol
    ro = dense.residual(pts, kid, kp, xo, b)
    rc = dense.residual(pts, kid, kp, x, b)
    assert rc <= 1.5 * ro + 1e-13


def test_cpp_tol_1e14_matches_dense_lu():
    pts, b = W.small_problem(d=2, n=2048, seed=8, nrhs=2)
    kid, kp = _paper_exp3(2048)
    x = CppAIFMM(pts, kid, kp, 32, 1e-14).factor().solve(b)
    xd = np.linalg.solve(dense.dense_matrix(pts, kid, kp), b)
    assert np.linalg.norm(x - xd) / np.linalg.norm(xd) <= 1e-12


def test_cpp_exact_redirection_solves_h2_matrix():
    """tol_c = 0: exact algebra on the NNCA matrix.  The densified NNCA matrix is written out
    by the numpy oracle (oracle/dense.py: h2_matrix) from the same skeletons (checked)."""
    for d, kind, kid, kp, n, leaf in ((2, "uniform_pm1", 0, (10.0, 0.0), 1500, 24),
                                      (2, "uniform_pm1", 1, (1.01, 0.1), 1500, 24),
                                      (3, "uniform_01", 2, (100.0, 0.0), 1200, 20)):
        pts, b = W.small_problem(d=d, n=n, kind=kind, seed=9)
        o = AIFMM(pts, kid, kp, leaf, 1e-5, tol_c=0.0)
        c = CppAIFMM(pts, kid, kp, leaf, 1e-5, tol_c=0.0)
        for l in range(2, c.L + 1):
            for bx in o.near[l]:
                assert np.array_equal(c.skeleton(l, bx), o.nnca.sk[l][bx])
        x = c.factor().solve(b)
        xh = np.linalg.solve(dense.h2_matrix(o), b)
        assert np.linalg.norm(x - xh) / np.linalg.norm(xh) <= 1e-11


def test_cpp_residual_monotone_in_tol():
    pts, b = W.small_problem(d=2, n=2048, seed=10)
    kid, kp = 0, (10.0, 0.0)
    res = [dense.residual(pts, kid, kp, CppAIFMM(pts, kid, kp, 32, tol).factor().solve(b), b)
           for tol in (1e-4, 1e-6, 1e-8, 1e-10, 1e-12)]
    assert all(a > b_ for a, b_ in zip(res, res[1:])), res


def test_cpp_zero_rhs_multi_rhs_and_threads_bit_identical():
    pts, b = W.small_problem(d=2, n=3000, seed=12, nrhs=3)
    c1 = CppAIFMM(pts, 0, (10.0, 0.0), 32, 1e-8, threads=1).factor()
    c4 = CppAIFMM(pts, 0, (10.0, 0.0), 32, 1e-8, threads=4).factor()
    assert np.all(c1.solve(np.zeros((3000, 2))) == 0.0)
    X1, X4 = c1.solve(b), c4.solve(b)
    assert np.array_equal(X1, X4)                                  # OpenMP: bit-identical
    for l in range(2, c1.L + 1):
        assert np.array_equal(c1.ranks(l, 1), c4.ranks(l, 1))
    for j in range(3):
        assert np.array_equal(X1[:, j], c1.solve(b[:, j]))          # columns are independent


def test_cpp_paper_exp3_first_row_golden(root):
    """tests/golden/paper_exp3_exp4.txt: Exp. 3 prints E_A = 2e-08 at N = 4900,
    eps_A = 1e-10 (2D 1/r, A_ii = sqrt(1000 N)); the C++ oracle must be at least as accurate."""
    rows = [l.split() for l in open(f"{root}/tests/golden/paper_exp3_exp4.txt") if l[0] != "#"]
    _, n, eps, ea = rows[0]
    n, eps, ea = int(n), float(eps), float(ea)
    pts = W.make_points("grid", n, 2, 0)
    b = W.make_rhs(n, 1, 0)
    kid, kp = _paper_exp3(n)
    x = CppAIFMM(pts, kid, kp, 64, eps).factor().solve(b)
    xd = np.linalg.solve(dense.dense_matrix(pts, kid, kp), b)
    e = np.linalg.norm(x - xd) / np.linalg.norm(xd)
    assert 1e-4 * eps <= e <= ea


def test_cpp_error_codes():
    with pytest.raises(OracleError) as e:
        CppAIFMM(np.zeros((5, 2)), 0, (1.0, 0.0), 2, 1e-8)          # coincident, log r
    assert e.value.code == -3
    p = np.zeros((4, 2))
    p[0, 0] = np.nan
    with pytest.raises(OracleError) as e:
        CppAIFMM(p, 0, (1.0, 0.0), 2, 1e-8)
    assert e.value.code == -2


def test_cpp_algorithm2_matches_numpy():
    """Alg. 2 (compress on creation, row f2) in the C++ oracle: same compression count as the
    numpy oracle's Alg. 2, solutions equal to rounding level."""
    pts, b = W.small_problem(d=2, n=3000, seed=13)
    o = AIFMM(pts, 0, (10.0, 0.0), 32, 1e-8, algorithm=2).factor()
    c = CppAIFMM(pts, 0, (10.0, 0.0), 32, 1e-8, algorithm=2).factor()
    assert c.stats()["compressions"] == o.stats["compressions"]
    x, xo = c.solve(b), o.solve(b)
    assert np.linalg.norm(x - xo) / np.linalg.norm(xo) <= 1e-7
