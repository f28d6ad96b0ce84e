"""GPU unit checks of the batched dense kernels behind the hot path, against plain numpy
float64 references: the Gauss-Jordan pivot inverse (reading R16) in its three variants —
shared-memory (n <= 160), blocked single-CTA panels, blocked 8-CTA cluster panels (few large
matrices: the top system) — on saddle-point matrices [[K, U], [V^T, 0]] that need pivoting; and the first stage of the
two-stage RRQR (reading R8b: R of a tall W^T) in each of its routes — one-CTA shared-memory
panels, TSQR row chunks over one or several rounds, one-CTA / cluster global-memory panels —
against numpy's Householder R (unique up to row signs) and the Gram identity R^T R = A^T A."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2301_12704_b200 import aifmm as G  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    G.load()
    yield


def _saddle(m, k, seed):
    rng = np.random.default_rng(seed)
    K = rng.standard_normal((m, m)) + 4 * np.eye(m)
    U = np.linalg.qr(rng.standard_normal((m, k)))[0]
    V = np.linalg.qr(rng.standard_normal((m, k)))[0]
    P = np.zeros((m + k, m + k))
    P[:m, :m], P[:m, m:], P[m:, :m] = K, U, V.T
    return P


@pytest.mark.parametrize("m,k", [(1, 0), (20, 13), (64, 60), (100, 61), (250, 90), (700, 300), (1100, 243)])
def test_pivot_inverse_matches_numpy(m, k):
    P = _saddle(m, k, m + k)
    Gi = G.debug_inverse(torch.from_numpy(P).cuda()).cpu().numpy()
    ref = np.linalg.inv(P)
    cond = np.linalg.cond(P)
    assert np.linalg.norm(Gi - ref) <= 1e-14 * cond * np.linalg.norm(ref) * np.sqrt(m + k)
    assert np.linalg.norm(P @ Gi - np.eye(m + k)) <= 1e-12 * cond


def test_singular_pivot_reported():
    P = _saddle(50, 10, 3)
    P[:, 7] = 0.0
    with pytest.raises(G.AIFMMError) as e:
        G.debug_inverse(torch.from_numpy(P).cuda())
    assert e.value.code == -5


@pytest.mark.parametrize("n,m,batch,rank", [
    (200, 16, 3, None),      # register panel, one row per thread
    (300, 40, 2, None),      # register panel, two rows per thread; two panels
    (700, 32, 2, None),      # TSQR: 2 chunks -> 64-row stack
    (700, 400, 1, None),     # no split (stack would not shrink): register panel on a 2-CTA cluster
    (2000, 64, 3, None),     # TSQR: 4 chunks -> 256-row stack
    (2000, 64, 2, 20),       # rank-deficient (fill-in-like), TSQR
    (5000, 100, 1, None),    # TSQR over three rounds (1000 -> 200 rows)
    (1700, 300, 2, None),    # TSQR rounds 1200 -> 900 -> 600, then shared-memory panels
    (1500, 500, 2, None),    # m > 384: one-CTA global-memory / cluster panels
    (6000, 450, 1, None),    # very long panels (cluster)
])
def test_tri_root_householder_and_tsqr(n, m, batch, rank):
    rng = np.random.default_rng(n + m)
    A = rng.standard_normal((batch, n, m))
    if rank is not None:
        A = np.einsum("bnr,brm->bnm", rng.standard_normal((batch, n, rank)), rng.standard_normal((batch, rank, m)))
    MT = G.debug_tri_root(torch.from_numpy(A).cuda()).cpu().numpy()   # (batch, m, r) = R^T
    for b in range(batch):
        R = MT[b].T
        r = min(n, m)
        assert R.shape == (r, m)
        assert np.all(np.tril(R, -1) == 0.0)
        nA = np.linalg.norm(A[b])
        # Gram identity (holds for any R of A, rank-deficient or not)
        assert np.linalg.norm(R.T @ R - A[b].T @ A[b]) <= 1e-13 * nA * nA
        if rank is None:   # full rank: R unique up to row signs
            Rn = np.linalg.qr(A[b], mode="r")
            D = np.sign(np.diag(R)) * np.sign(np.diag(Rn))
            assert np.linalg.norm(D[:, None] * R - Rn) <= 1e-12 * nA


def test_tri_root_shared_memory_panel_variant():
    """The one-CTA shared-memory panel (routing variant AIFMM_HH_SMEM=1, read once per process, so
    it runs in a subprocess) against numpy's R on 512 < n <= 768 panels."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, torch, sys; sys.path.insert(0, %r)\n"
        "from paper_2301_12704_b200 import aifmm as G\n"
        "rng = np.random.default_rng(7)\n"
        "for n, m in ((700, 400), (760, 300)):\n"
        "    A = rng.standard_normal((2, n, m))\n"
        "    R = G.debug_tri_root(torch.from_numpy(A).cuda()).cpu().numpy()\n"
        "    for b in range(2):\n"
        "        Rg = R[b].T; Rn = np.linalg.qr(A[b], mode='r')\n"
        "        D = np.sign(np.diag(Rg)) * np.sign(np.diag(Rn))\n"
        "        assert np.linalg.norm(D[:, None] * Rg - Rn) <= 1e-12 * np.linalg.norm(A[b]), (n, m)\n"
        "print('ok')\n" % os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    env = dict(os.environ, AIFMM_HH_SMEM="1", AIFMM_TSQR_MMAX="0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("cl", [2, 4])
def test_pivot_inverse_cluster_sizes(cl):
    """The Gauss-Jordan cluster panel with 2- and 4-CTA clusters (chosen for larger batches;
    forced here through AIFMM_GJ_CL, read once per process, so it runs in a subprocess)."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, torch, sys; sys.path.insert(0, %r)\n"
        "from paper_2301_12704_b200 import aifmm as G\n"
        "def saddle(m, k, seed):\n"
        "    rng = np.random.default_rng(seed)\n"
        "    K = rng.standard_normal((m, m)) + 4 * np.eye(m)\n"
        "    U = np.linalg.qr(rng.standard_normal((m, k)))[0]\n"
        "    V = np.linalg.qr(rng.standard_normal((m, k)))[0]\n"
        "    P = np.zeros((m + k, m + k)); P[:m, :m], P[:m, m:], P[m:, :m] = K, U, V.T\n"
        "    return P\n"
        "for m, k in ((250, 90), (700, 300)):\n"
        "    P = saddle(m, k, 3)\n"
        "    Gi = G.debug_inverse(torch.from_numpy(P).cuda()).cpu().numpy()\n"
        "    cond = np.linalg.cond(P)\n"
        "    assert np.linalg.norm(P @ Gi - np.eye(m + k)) <= 1e-12 * cond, (m, k)\n"
        "print('ok')\n" % os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    env = dict(os.environ, AIFMM_GJ_CL=str(cl))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("env", [{"AIFMM_SYM_SCHUR": "1"}, {"AIFMM_NULLSPACE": "1"}, {"AIFMM_NULLSPACE": "0"},
                                 {"AIFMM_SYM_SCHUR": "1", "AIFMM_NULLSPACE": "1"}],
                         ids=["R30", "R31-all", "R31-off", "R30+R31-all"])
def test_opt_in_elimination_variants(env):
    """The opt-in elimination variants (read once per process, so each runs in a subprocess):
    R30 symmetric Schur pairs, R31 null-space pivot inverses with rank-(m-k) Schur terms.  Both
    are exact in exact arithmetic, so the factorization must agree with the oracle exactly as the
    default does: solution within 10*tol, residual within 2x, on a ragged 2D log case and a 3D
    1/r case; and with tol_c = 0 the solve must equal the densified NNCA matrix's."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import numpy as np, torch, sys; sys.path.insert(0, %r)\n"
        "from paper_2301_12704_b200 import aifmm as G, workloads as W\n"
        "from oracle.factor import AIFMM as Oracle\n"
        "from oracle import dense\n"
        "for kind, n, d, kid, kp, leaf, tol in (('uniform_pm1', 3000, 2, 0, (10.0, 0.0), 40, 1e-8),\n"
        "                                       ('uniform_01', 3000, 3, 2, (100.0, 0.0), 32, 1e-7)):\n"
        "    pts = W.make_points(kind, n, d, 21); b = W.make_rhs(n, 2, 21)\n"
        "    xo = Oracle(pts, kid, kp, leaf, tol).factor().solve(b)\n"
        "    G.free(); G.build(torch.from_numpy(pts).cuda(), kid, kp, leaf, tol); G.factor()\n"
        "    x = G.solve(torch.from_numpy(b).cuda()).cpu().numpy()\n"
        "    rel = np.linalg.norm(x - xo) / np.linalg.norm(xo)\n"
        "    assert rel <= 10 * tol, (kind, rel)\n"
        "    assert dense.residual(pts, kid, kp, x, b) <= 2 * dense.residual(pts, kid, kp, xo, b) + 1e-13\n"
        "pts, b = W.small_problem(d=2, n=1500, seed=9)\n"
        "o = Oracle(pts, 0, (10.0, 0.0), 24, 1e-5, tol_c=0.0)\n"
        "G.free(); G.set_compression_tol(0.0); G.build(torch.from_numpy(pts).cuda(), 0, (10.0, 0.0), 24, 1e-5); G.factor()\n"
        "x = G.solve(torch.from_numpy(b).cuda()).cpu().numpy()\n"
        "xh = np.linalg.solve(dense.h2_matrix(o), b)\n"
        "assert np.linalg.norm(x - xh) / np.linalg.norm(xh) <= 1e-10\n"
        "print('ok')\n" % root)
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True,
                       timeout=900, cwd=root)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]


@pytest.mark.parametrize("m,k,batch", [(150, 40, 5), (250, 90, 7), (333, 1, 3), (700, 300, 2)])
def test_fused_gauss_jordan_matches_panel_path(m, k, batch):
    """The fused one-CTA-per-matrix Gauss-Jordan (panel steps + in-kernel DMMA updates, one
    launch) against the panel-launch + GEMM-launch path on the same saddle-point matrices:
    bitwise identical (same pivots, same DMMA k order, C + acc with beta = 1), and an inverse
    to the numpy bar; ragged last panel (n not a multiple of 32) and n > one update tile."""
    n = m + k
    Ps = np.stack([_saddle(m, k, 100 + t) for t in range(batch)])
    T = torch.from_numpy(Ps).cuda()
    old = G.debug_inverse_batch(T.clone(), path=1).cpu().numpy()
    new = G.debug_inverse_batch(T.clone(), path=2).cpu().numpy()
    assert np.array_equal(old, new)
    for t in range(batch):
        cond = np.linalg.cond(Ps[t])
        assert np.linalg.norm(Ps[t] @ new[t] - np.eye(n)) <= 1e-12 * cond


def test_fused_gauss_jordan_singular_reported():
    Ps = np.stack([_saddle(180, 20, 7 + t) for t in range(3)])
    Ps[1][:, 50] = 0.0
    with pytest.raises(G.AIFMMError) as e:
        G.debug_inverse_batch(torch.from_numpy(Ps).cuda(), path=2)
    assert e.value.code == -5
