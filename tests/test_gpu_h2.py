"""GPU parity for row a8 (BASELINE config 5): the H2 matvec and AIFMM-preconditioned GMRES
through the C-ABI against oracle/h2.py on the same seeded inputs.

Bars: the matvec uses the same integer NNCA decisions as the oracle (ranks bit-exact), so the
products agree to rounding (1e-11 relative); GMRES reaches the requested relative residual, in
at most one iteration more than the oracle, and its solution agrees with the oracle's within
the stopping tolerance amplified by the matrix condition (checked through the exact residual).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import dense                          # noqa: E402
from oracle.factor import AIFMM as Oracle          # noqa: E402
from oracle.h2 import H2, gmres                    # noqa: E402
from paper_2301_12704_b200 import aifmm as G       # noqa: E402
from paper_2301_12704_b200 import workloads as W   # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    G.load()
    yield
    G.free()


@pytest.mark.parametrize("d,kind,kid,kp,n,leaf,tol", [
    (2, "uniform_pm1", 0, (10.0, 0.0), 3000, 32, 1e-10),
    (3, "uniform_01", 2, (100.0, 0.0), 3000, 32, 1e-10),
    (2, "uniform_pm1", 1, (1.01, 0.1), 2500, 24, 1e-8),
])
def test_h2_matvec_parity(d, kind, kid, kp, n, leaf, tol):
    pts = W.make_points(kind, n, d, 40)
    x = W.make_rhs(n, 3, 40)
    h = H2(pts, kid, kp, leaf, tol)
    yo = h.matvec(x)
    G.free()
    G.build(torch.from_numpy(pts).cuda(), kid, kp, leaf, 0.5)
    G.matvec_build(tol)
    y = G.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.linalg.norm(y - yo) <= 1e-11 * np.linalg.norm(yo)
    y1 = G.matvec(torch.from_numpy(np.ascontiguousarray(x[:, 1])).cuda()).cpu().numpy()
    assert np.abs(y1 - y[:, 1]).max() <= 1e-13 * np.abs(y[:, 1]).max()


def test_gmres_preconditioned_parity_config5_style():
    n = 3000
    pts = W.make_points("uniform_01", n, 3, 41)
    b = W.make_rhs(n, 1, 41)[:, 0]
    kp = (100.0, 0.0)
    h = H2(pts, 2, kp, 32, 1e-10)
    P = Oracle(pts, 2, kp, 32, 1e-3).factor()
    xo, ito, rro = gmres(h.matvec, b, precond=P.solve, restart=30, rtol=1e-10)
    G.free()
    G.build(torch.from_numpy(pts).cuda(), 2, kp, 32, 1e-3)
    G.factor()
    G.matvec_build(1e-10)
    x, it, rr = G.gmres(torch.from_numpy(b).cuda(), restart=30, rtol=1e-10, maxit=200, precond=True)
    x = x.cpu().numpy()
    assert rr <= 1e-10 and rro <= 1e-10
    assert abs(it - ito) <= 1
    A = dense.dense_matrix(pts, 2, kp)
    assert np.linalg.norm(A @ x - b) <= 1e-8 * np.linalg.norm(b)
    assert np.linalg.norm(x - xo) <= 1e-7 * np.linalg.norm(xo)
    # unpreconditioned GMRES needs more iterations on the same system
    _, it0, rr0 = G.gmres(torch.from_numpy(b).cuda(), restart=30, rtol=1e-10, maxit=it, precond=False)
    assert rr0 > 1e-10


def test_gmres_three_preconditioners_parity():
    """Row f3 (the paper's comparison I_G / I_BD / I_pA, table) on a
    config-5-style 3D 1/r problem: GMRES with no preconditioner, the leaf block-diagonal inverse
    and the AIFMM(1e-3) factor.  Each GPU iteration count is within one of the oracle's with the
    same preconditioner, and the counts are ordered I_pA < I_BD <= I_G."""
    n = 3000
    pts = W.make_points("uniform_01", n, 3, 43)
    b = W.make_rhs(n, 1, 43)[:, 0]
    kp = (100.0, 0.0)
    from oracle.h2 import block_diagonal_precond
    h = H2(pts, 2, kp, 32, 1e-10)
    P = Oracle(pts, 2, kp, 32, 1e-3).factor()
    bd = block_diagonal_precond(P.tree, 2, kp)
    G.free()
    G.build(torch.from_numpy(pts).cuda(), 2, kp, 32, 1e-3)
    G.factor()
    G.matvec_build(1e-10)
    its, res = {}, {}
    for name, pre_o, pre_g in (("G", None, 0), ("BD", bd, 2), ("pA", P.solve, 1)):
        _, ito, rro = gmres(h.matvec, b, precond=pre_o, restart=30, rtol=1e-10, maxit=120)
        _, it, rr = G.gmres(torch.from_numpy(b).cuda(), restart=30, rtol=1e-10, maxit=120, precond=pre_g)
        if rro <= 1e-10:                      # converged: iteration counts within one
            assert rr <= 1e-10 and abs(it - ito) <= 1, (name, it, ito, rr)
        else:                                 # not converged in 120: same residual history
            assert it == ito == 120 and abs(rr - rro) <= 0.05 * rro, (name, rr, rro)
        its[name], res[name] = it, rr
    # the paper's ordering I_pA << I_BD, I_G: the AIFMM preconditioner converges first
    print(f"GMRES iterations (relative residual): {its} {res}")
    assert res["pA"] <= 1e-10 and its["pA"] < its["BD"] and its["pA"] < its["G"], (its, res)
