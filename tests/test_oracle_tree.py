"""Pins for oracle/tree.py against the paper's definitions (not against itself)."""
import itertools

import numpy as np
import pytest

from oracle.tree import Tree, build_lists, greedy_colours, chebyshev, admissible_geometric, root_box
from paper_2301_12704_b200 import workloads as W


def test_root_box_examples():
    # symmetric extremes; (-1,0),(2,0) -> centre (0.5,0), half side 1.5
    g, two_h = root_box(np.array([[-1.0, -1.0], [1.0, 1.0]]))
    assert np.allclose(g, [-1, -1]) and two_h == 2.0
    g, two_h = root_box(np.array([[-1.0, 0.0], [2.0, 0.0]]))
    assert np.allclose(g, [-1.0, -1.5]) and two_h == 3.0


@pytest.mark.parametrize("d,n,nmax,kind", [(2, 2048, 32, "uniform_pm1"), (3, 3000, 40, "uniform_01"),
                                            (2, 4096, 64, "grid")])
def test_tree_membership_bruteforce(d, n, nmax, kind):
    pts = W.make_points(kind, n, d, 11)
    t = Tree(pts, nmax)
    assert t.L >= 2
    # P:123 every leaf holds <= n_max points; L minimal (depth L-1 violates unless L == 2)
    leaf_counts = np.diff(t.off[t.L])
    assert leaf_counts.max() <= nmax
    # brute-force box membership from geometry: point p lies in the box whose
    # half-open cell [g + 2h*k/2^L, g + 2h*(k+1)/2^L) contains it
    lo = t.g
    side = t.two_h / (1 << t.L)
    for j in range(0, n, max(1, n // 300)):
        p = t.points[j]
        leaf = int(np.searchsorted(t.off[t.L], j, side="right") - 1)
        c = t.coords(t.L, leaf)
        for a in range(d):
            x0 = lo[a] + side * c[a]
            assert x0 - 1e-12 <= p[a] <= x0 + side + 1e-12
    # partition: every level's offsets cover all points once
    for l in range(t.L + 1):
        assert t.off[l][0] == 0 and t.off[l][-1] == n
        assert np.all(np.diff(t.off[l]) >= 0)
    # perm is a permutation
    assert np.array_equal(np.sort(t.perm), np.arange(n))
    if t.L > 2:
        lk = t.sorted_leaf_key >> d
        _, cnt = np.unique(lk, return_counts=True)
        assert cnt.max() > nmax


def test_grid_configs_have_exact_leaf_size():
    # BASELINE configs 1 and 4: 64 points per leaf at L = 3 (2D) / L = 4 (3D) under the <= rule
    t = Tree(W.make_points("grid", 4096, 2, 0), 64)
    assert t.L == 3 and set(np.diff(t.off[3])) == {64}
    t = Tree(W.make_points("grid", 16 ** 3, 3, 0), 64)
    assert t.L == 2 and set(np.diff(t.off[2])) == {64}


def test_lists_counts_and_symmetry():
    t = Tree(W.make_points("grid", 64 * 64, 2, 0), 4)   # L = 5, full grid
    near, il = build_lists(t)
    for l in near:
        side = 1 << l
        for b in near[l]:
            c = t.coords(l, b)
            interior = all(2 <= x < side - 2 for x in c)
            if interior:
                assert len(near[l][b]) == 9
                if l >= 3 and all(4 <= x < side - 4 for x in c):
                    assert len(il[l][b]) == 27
            if all(x in (0, side - 1) for x in c):
                assert len(near[l][b]) == 4          # corner box
            for j in near[l][b]:
                assert b in near[l][j]
            for j in il[l][b]:
                assert b in il[l][j]
                assert j not in near[l][b]


def test_lists_3d_interior_counts():
    t = Tree(W.make_points("grid", 16 ** 3, 3, 0), 1)   # L = 4
    near, il = build_lists(t)
    l = 4
    b = t.box_id((7, 7, 7), l)
    assert len(near[l][b]) == 27 and len(il[l][b]) == 189


def test_admissibility_equals_chebyshev_and_coverage():
    pts, _ = W.small_problem(d=2, n=1500, seed=2)
    t = Tree(pts, 12)
    near, il = build_lists(t)
    for l in near:
        boxes = sorted(near[l])
        for a, b in itertools.product(boxes, boxes):
            # Eq. adm_condn on geometry == Chebyshev index distance >= 2 (R5)
            assert admissible_geometric(t, l, a, b) == (chebyshev(t, l, a, b) >= 2)
            assert (b in near[l][a]) == (not admissible_geometric(t, l, a, b))
    # completeness: every pair of leaves is covered exactly once by a leaf near pair or an
    # IL pair of ancestors at exactly one level (FMM structure Eqs.)
    L = t.L
    leaves = sorted(near[L])
    for a, b in itertools.product(leaves, leaves):
        hits = int(b in near[L][a])
        for l in range(2, L + 1):
            aa, bb = a >> (t.d * (L - l)), b >> (t.d * (L - l))
            hits += int(bb in il[l].get(aa, []))
        assert hits == 1, (a, b)


def test_colouring_valid_and_parity_on_full_grid():
    t = Tree(W.make_points("grid", 64 * 64, 2, 0), 4)
    near, _ = build_lists(t)
    for l in near:
        col = greedy_colours(t, near[l])
        for b in near[l]:
            for j in near[l][b]:
                if j != b:
                    assert col[j] != col[b]
            c = t.coords(l, b)
            assert col[b] == (c[0] % 2) + 2 * (c[1] % 2)    # parity colouring (4 colours)
    t3 = Tree(W.make_points("grid", 8 ** 3, 3, 0), 1)
    near3, _ = build_lists(t3)
    col = greedy_colours(t3, near3[3])
    assert max(col.values()) == 7
