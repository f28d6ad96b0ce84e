"""GPU parity: the CUDA path (through the C-ABI) against the oracle on the same seeded inputs.

Bars (BASELINE.json north_star): integer outputs (tree permutation, box offsets, N/IL lists,
colours, NNCA ranks) bit-exact; solution within 10*tol relative 2-norm of the oracle's;
relative residual (exact direct sum, 4096 sampled rows at large N) within 2x the oracle's.
"""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import dense                      # noqa: E402
from oracle.factor import AIFMM as Oracle     # noqa: E402
from paper_2301_12704_b200 import aifmm as G  # noqa: E402
from paper_2301_12704_b200 import workloads as W  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    G.load()
    yield
    G.free()


def _gpu_solve(pts, b, kid, kp, leaf, tol, tol_c=None):
    G.free()
    if tol_c is not None:
        G.set_compression_tol(tol_c)
    G.build(torch.from_numpy(pts).cuda(), kid, kp, leaf, tol)
    G.factor()
    return G.solve(torch.from_numpy(np.ascontiguousarray(b)).cuda()).cpu().numpy()


def _integer_parity(o, d):
    perm, L = G.get_tree(o.tree.n)
    assert L == o.tree.L
    assert np.array_equal(perm, o.tree.perm)
    for l in range(0, L + 1):
        assert np.array_equal(G.get_level_offsets(l, d), o.tree.off[l])
    for l in range(2, L + 1):
        nptr, nidx, iptr, iidx = G.get_lists(l, d)
        col = G.get_colours(l, d)
        rk = G.get_ranks(l, d, 0)
        nb = 1 << (d * l)
        for b in range(nb):
            if b in o.near[l]:
                assert list(nidx[nptr[b]:nptr[b + 1]]) == o.near[l][b]
                assert list(iidx[iptr[b]:iptr[b + 1]]) == o.il[l][b]
                assert col[b] == o.colour[l][b]
                assert rk[b] == o.nnca.rank(l, b)
            else:
                assert nptr[b + 1] == nptr[b] and col[b] == -1
        # NNCA skeletons and far pivots (row a3): the same indices in the same pivot order
        skp, sk, fp = G.get_skeletons(l, d)
        for b in o.nnca.sk[l]:
            assert list(sk[skp[b]:skp[b + 1]]) == o.nnca.sk[l][b].tolist(), (l, b)
            assert list(fp[skp[b]:skp[b + 1]]) == o.nnca.fp[l][b].tolist(), (l, b)


CASES = [
    # (name, points kind, n, d, kernel, kparams, leaf, tol, nrhs)
    ("cfg1_grid_log", "grid", 4096, 2, 0, (10.0, 0.0), 64, 1e-8, 1),
    ("rand2d_log_ragged", "uniform_pm1", 3000, 2, 0, (10.0, 0.0), 40, 1e-8, 2),
    ("rand2d_matern", "uniform_pm1", 2500, 2, 1, (1.01, 0.1), 32, 1e-6, 1),
    ("rand2d_invr", "uniform_pm1", 2048, 2, 2, (float(np.sqrt(1000 * 2048)), 0.0), 32, 1e-10, 3),
    ("rand3d_invr", "uniform_01", 3000, 3, 2, (100.0, 0.0), 32, 1e-7, 1),
    ("grid3d_invr", "grid", 4096, 3, 2, (128.0, 0.0), 64, 1e-7, 2),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_parity_small(case):
    name, kind, n, d, kid, kp, leaf, tol, nrhs = case
    pts = W.make_points(kind, n, d, 21)
    b = W.make_rhs(n, nrhs, 21)
    o = Oracle(pts, kid, kp, leaf, tol).factor()
    xo = o.solve(b)
    x = _gpu_solve(pts, b, kid, kp, leaf, tol)
    _integer_parity(o, d)
    rel = np.linalg.norm(x - xo) / np.linalg.norm(xo)
    assert rel <= 10 * tol, rel
    ro = dense.residual(pts, kid, kp, xo, b)
    rg = dense.residual(pts, kid, kp, x, b)
    assert rg <= 2 * ro + 1e-13, (rg, ro)      # 1e-13: rounding-noise floor


def test_exact_redirection_matches_densified_nnca():
    """tol_c = 0: the GPU elimination is exact algebra on the NNCA matrix (same integer
    decisions as the oracle, so the same densified H2 matrix)."""
    pts, b = W.small_problem(d=2, n=1500, seed=9)
    o = Oracle(pts, 0, (10.0, 0.0), 24, 1e-5, tol_c=0.0)
    x = _gpu_solve(pts, b, 0, (10.0, 0.0), 24, 1e-5, tol_c=0.0)
    xh = np.linalg.solve(dense.h2_matrix(o), b)
    assert np.linalg.norm(x - xh) / np.linalg.norm(xh) <= 1e-10
    G.set_compression_tol(1e-5)


def test_multi_rhs_equals_columns_and_zero_rhs():
    pts, b = W.small_problem(d=2, n=2000, seed=12, nrhs=4)
    G.free()
    G.build(torch.from_numpy(pts).cuda(), 0, (10.0, 0.0), 32, 1e-8)
    G.factor()
    X = G.solve(torch.from_numpy(b).cuda()).cpu().numpy()
    for j in range(4):
        xj = G.solve(torch.from_numpy(np.ascontiguousarray(b[:, j])).cuda()).cpu().numpy()
        assert np.abs(X[:, j] - xj).max() <= 1e-12 * np.abs(xj).max()
    z = G.solve(torch.zeros(2000, 2, dtype=torch.float64, device="cuda")).cpu().numpy()
    assert np.all(z == 0.0)
    # repeated solves do not alter the factorization
    X2 = G.solve(torch.from_numpy(b).cuda()).cpu().numpy()
    assert np.array_equal(X, X2)
    # the binding never overwrites the caller's right-hand side (one and several columns)
    b1 = torch.from_numpy(np.ascontiguousarray(b[:, 0])).cuda()
    keep = b1.clone()
    G.solve(b1)
    assert torch.equal(b1, keep)
    # end-to-end host path gives the same numbers
    Xh = G.solve_host(b)
    assert np.abs(Xh - X).max() <= 1e-13 * np.abs(X).max()


@pytest.mark.parametrize("n", [1, 2, 7, 65])
def test_tiny_inputs(n):
    """Degenerate trees: one point, a few points (empty IL, rank-0 boxes, empty boxes)."""
    pts, b = W.small_problem(d=2, n=n, seed=30 + n)
    kp = (5.0 + n, 0.0)
    o = Oracle(pts, 2, kp, 4, 1e-8).factor()
    xo = o.solve(b)
    x = _gpu_solve(pts, b, 2, kp, 4, 1e-8)
    _integer_parity(o, 2)
    assert np.linalg.norm(x - xo) <= 1e-12 * max(np.linalg.norm(xo), 1e-300)
    A = dense.dense_matrix(pts, 2, kp)
    assert np.linalg.norm(A @ x - b) <= 1e-7 * np.linalg.norm(b)


def test_error_codes():
    G.free()
    p = torch.zeros(4, 2, dtype=torch.float64, device="cuda")
    with pytest.raises(G.AIFMMError) as e:          # more coincident points than a leaf holds
        G.build(p, 0, (1.0, 0.0), 2, 1e-6)
    assert e.value.code == -3
    with pytest.raises(G.AIFMMError) as e:          # coincident points, singular kernel
        G.build(p, 0, (1.0, 0.0), 4, 1e-6)
        G.factor()
    assert e.value.code == -3
    p = torch.tensor([[0.0, 0.0], [float("nan"), 1.0]], dtype=torch.float64, device="cuda")
    with pytest.raises(G.AIFMMError) as e:
        G.build(p, 0, (1.0, 0.0), 2, 1e-6)
    assert e.value.code == -2
    with pytest.raises(G.AIFMMError) as e:
        G.build(torch.zeros(4, 2, dtype=torch.float64, device="cuda"), 0, (1.0, 0.0), 2, 2.0)
    assert e.value.code == -1
    G.free()
    with pytest.raises(G.AIFMMError) as e:
        G.factor()
    assert e.value.code == -6
    with pytest.raises(G.AIFMMError) as e:
        G.solve(torch.zeros(4, dtype=torch.float64, device="cuda"))
    assert e.value.code == -6


@pytest.fixture(scope="module")
def cfg2_run():
    """BASELINE config 2 at full size (N = 65536, 16 RHS, tol 1e-10) in the configuration
    bench.py --cfg 2 times: GPU and numpy-oracle solutions, sampled direct-sum residuals (4096
    rows) and final ranks, computed once for the tests below."""
    cfg = W.CONFIGS[1]
    pts, b = W.make(cfg)
    o = Oracle(pts, cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol).factor()
    xo = o.solve(b)
    x = _gpu_solve(pts, b, cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol)
    rows = W.residual_rows(cfg.n, cfg.seed)
    ro = dense.residual(pts, cfg.kernel_id, cfg.kparams, xo, b, rows)
    rg = dense.residual(pts, cfg.kernel_id, cfg.kparams, x, b, rows)
    rel = float(np.linalg.norm(x - xo) / np.linalg.norm(xo))
    gr = {l: G.get_ranks(l, 2, 1) for l in o.levels}
    mism = {l: int(sum(1 for bx in o.levels[l].boxes if gr[l][bx] != o.levels[l].k[bx])) for l in o.levels}
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cfg2_oracle_rounding_floor.json")))
    print(f"config 2: rel solution diff {rel:.3e} (oracle vs itself {g['same_decisions_rel_solution_diff']:.2e}), "
          f"residual {rg:.3e} (oracle {ro:.3e}), final-rank mismatches {mism} "
          f"(oracle vs itself: {g['free_decisions_rank_mismatches']})")
    return dict(cfg=cfg, rel=rel, rg=rg, ro=ro, mism=mism, golden=g)


def test_config2_full_size_residual(cfg2_run):
    """North_star bar 2 on config 2: sampled direct-sum residual within 2x the oracle's."""
    r = cfg2_run
    assert r["rg"] <= 2 * r["ro"], (r["rg"], r["ro"])


def test_config2_full_size_solution_north_star_bar(cfg2_run):
    """North_star bar 1 as stated: solution within 10*tol of the oracle's, a hard gate (the GPU
    path is bitwise deterministic and lands at 6.6e-10).  Reading R24 records that
    the oracle itself spreads 2.2e-9 under exact-arithmetic-equivalent rounding changes on this
    workload, so a kernel change that alters rounding may move this number; such a change
    has to keep it below 1e-9 or be reverted."""
    r = cfg2_run
    assert r["rel"] <= 10 * r["cfg"].tol, r["rel"]


def test_config2_full_size_solution_rounding_floor(cfg2_run):
    """Reading R24 reported separately: the solution lies within the spread the oracle itself
    shows under exact-arithmetic-equivalent rounding changes (1.5x that floor).  Final ranks are
    reported by the fixture, not gated: the oracle against itself with free decisions already
    differs in ~110 boxes."""
    r = cfg2_run
    floor = r["golden"]["same_decisions_rel_solution_diff"]
    assert r["rel"] <= max(10 * r["cfg"].tol, 1.5 * floor), (r["rel"], floor)


def test_gpu_residual_matches_oracle_direct_sum():
    """Row a9 on the GPU (aifmm_residual): the direct-sum relative residual of a solution equals
    the oracle's (oracle/dense.py: residual) on all rows and on a sampled row set, for every
    kernel (several 128-row blocks, a ragged last block, several source chunks)."""
    for kid, kp, d, kind in ((0, (10.0, 0.0), 2, "uniform_pm1"), (1, (1.01, 0.1), 2, "uniform_pm1"),
                             (2, (100.0, 0.0), 3, "uniform_01")):
        pts, b = W.small_problem(d=d, n=2900, kind=kind, seed=40 + kid, nrhs=3)
        G.free()
        G.build(torch.from_numpy(pts).cuda(), kid, kp, 40, 1e-6)
        G.factor()
        X = G.solve(torch.from_numpy(b).cuda())
        x = X.cpu().numpy()
        rows = np.sort(np.random.default_rng(kid).choice(2900, 700, replace=False))
        for rr in (None, rows):
            ro = dense.residual(pts, kid, kp, x, b, rr)
            rg = G.residual(X, torch.from_numpy(b).cuda(), rr)
            assert abs(rg - ro) <= 1e-9 * ro + 1e-13, (kid, rg, ro)   # 1e-13: rounding floor of A x - b
        # an exact solution of a perturbed system: residual of (X, A X) is ~0
        Y = torch.from_numpy(dense.dense_matrix(pts, kid, kp) @ x).cuda()
        assert G.residual(X, Y) <= 1e-13


@pytest.mark.parametrize("case", CASES[:2] + CASES[4:5], ids=[c[0] for c in CASES[:2] + CASES[4:5]])
def test_algorithm2_parity(case):
    """Row f2: Algorithm 2 (compress on creation) on the GPU (aifmm_set_algorithm(2))
    against the oracle's Algorithm 2: the number of compressions within 2% (it depends on the
    rank decisions through R28: a box whose compression fills its basis makes no further
    fill-in), solution within 10*tol, residual within 2x."""
    name, kind, n, d, kid, kp, leaf, tol, nrhs = case
    pts = W.make_points(kind, n, d, 21)
    b = W.make_rhs(n, nrhs, 21)
    o = Oracle(pts, kid, kp, leaf, tol, algorithm=2).factor()
    xo = o.solve(b)
    G.set_algorithm(2)
    try:
        G.reset_counters()
        x = _gpu_solve(pts, b, kid, kp, leaf, tol)
        st = G.stats()
    finally:
        G.set_algorithm(3)
    assert abs(int(st["compressions"]) - o.stats["compressions"]) <= max(2, 0.02 * o.stats["compressions"])
    assert np.linalg.norm(x - xo) / np.linalg.norm(xo) <= 10 * tol
    assert dense.residual(pts, kid, kp, x, b) <= 2 * dense.residual(pts, kid, kp, xo, b) + 1e-13


def _golden(name):
    p = os.path.join(os.path.dirname(__file__), "golden", f"{name}_oracle.npz")
    if not os.path.exists(p):
        pytest.skip(f"{p} not generated (tools/oracle_golden.py)")
    g = np.load(p)
    return g, json.loads(str(g["meta"]))


def test_config3_full_size_parity():
    """BASELINE config 3 at full size (N = 2^20 Matern, leaf 128, tol 1e-8, 1 RHS) in the
    configuration bench.py times, against the serial C++ oracle's cached result
    (tests/golden/cfg3_rand2d_matern_1M_oracle.npz, written by tools/oracle_golden.py on a GPU
    box's host): integer outputs (tree, lists, colours, NNCA ranks) bit-exact with the C++
    oracle's build (re-run here), solution within 10*tol of the oracle's, sampled direct-sum
    residual within 2x the oracle's."""
    from oracle.cpp import CppAIFMM
    cfg = W.CONFIGS[2]
    g, meta = _golden(cfg.name)
    pts, b = W.make(cfg)
    G.free()
    G.build(torch.from_numpy(pts).cuda(), cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol)
    c = CppAIFMM(pts, cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol, threads=os.cpu_count() or 1)
    perm, L = G.get_tree(cfg.n)
    assert L == c.L == meta["L"]
    assert np.array_equal(perm, c.perm())
    for l in range(2, L + 1):
        assert np.array_equal(G.get_level_offsets(l, 2), c.offsets(l))
        gn = G.get_lists(l, 2)
        cn = c.lists(l)
        for a, bb in zip(gn, cn):
            assert np.array_equal(a, bb)
        assert np.array_equal(G.get_colours(l, 2), c.colours(l))
        assert np.array_equal(G.get_ranks(l, 2, 0), g[f"nnca_{l}"])
        skp, sk, _ = G.get_skeletons(l, 2)
        for bx in np.flatnonzero(np.diff(skp)):
            assert np.array_equal(sk[skp[bx]:skp[bx + 1]], c.skeleton(l, int(bx))), (l, bx)
    del c
    G.factor()
    X = G.solve(torch.from_numpy(np.ascontiguousarray(b)).cuda())
    x = X.cpu().numpy()
    xo = g["x"]
    rel = np.linalg.norm(x - xo) / np.linalg.norm(xo)
    rows = W.residual_rows(cfg.n, cfg.seed)
    rg = G.residual(X, torch.from_numpy(np.ascontiguousarray(b)).cuda(), rows)
    ro = meta["residual_4096_rows"]
    mism = {l: int(np.sum(G.get_ranks(l, 2, 1) != g[f"ranks_{l}"])) for l in range(2, L + 1)}
    print(f"config 3: rel solution diff {rel:.3e}, residual {rg:.3e} (oracle {ro:.3e}), final-rank mismatches {mism}")
    assert rg <= 2 * ro, (rg, ro)
    assert rel <= 10 * cfg.tol, (rel, mism)


@pytest.mark.parametrize("ci,n", [(4, 32768), (5, 65536)], ids=["cfg4_grid3d_32768", "cfg5_rand3d_65536"])
def test_reduced_config_parity_against_cpp_oracle(ci, n):
    """BASELINE configs 4 and 5 at reduced N (config 4: the 32^3 grid instead of 64^3, which does
    not fit one GPU; config 5: 65536 of its 2^21 points, the AIFMM(1e-3) preconditioner applied
    to b) with the config's kernel, diagonal, leaf size and tol, against the serial C++ oracle's
    cached result (tools/oracle_golden.py): NNCA ranks bit-exact, solution within 10*tol of the
    oracle's, sampled direct-sum residual within 2x."""
    cfg = W.CONFIGS[ci - 1]
    g, meta = _golden(f"{cfg.name}_n{n}")
    pts, b = W.make(cfg, n=n)
    G.free()
    G.build(torch.from_numpy(pts).cuda(), cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol)
    perm, L = G.get_tree(n)
    assert L == meta["L"]
    for l in range(2, L + 1):
        assert np.array_equal(G.get_ranks(l, cfg.d, 0), g[f"nnca_{l}"])
    G.factor()
    Bd = torch.from_numpy(np.ascontiguousarray(b)).cuda()
    X = G.solve(Bd)
    x = X.cpu().numpy()
    xo = g["x"]
    rel = np.linalg.norm(x - xo) / np.linalg.norm(xo)
    rg = G.residual(X, Bd, W.residual_rows(n, cfg.seed))
    ro = meta["residual_4096_rows"]
    print(f"{cfg.name} N={n}: rel solution diff {rel:.3e}, residual {rg:.3e} (oracle {ro:.3e})")
    assert rg <= 2 * ro, (rg, ro)
    assert rel <= 10 * cfg.tol, rel


def test_factorization_deterministic():
    """Two factorizations of the same input give bitwise-identical solutions and final ranks:
    every reduction of the GPU path has a fixed order (no atomics), and the host planning is
    deterministic."""
    pts, b = W.small_problem(d=2, n=6000, seed=17, nrhs=2)
    out = []
    for _ in range(2):
        G.free()
        G.build(torch.from_numpy(pts).cuda(), 1, (1.01, 0.1), 48, 1e-8)
        G.factor()
        x = G.solve(torch.from_numpy(b).cuda()).cpu().numpy()
        perm, L = G.get_tree(6000)
        out.append((x, [G.get_ranks(l, 2, 1) for l in range(2, L + 1)]))
    assert np.array_equal(out[0][0], out[1][0])
    assert all(np.array_equal(a, c) for a, c in zip(out[0][1], out[1][1]))
