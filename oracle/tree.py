"""Tree, lists and colouring (oracle; test infrastructure only).

P:121-123 (§2.1): the root is the smallest hypercube containing the points; a
uniform 2^d tree is refined until every box holds no more than n_max points.
P:198-230 (§2.2): strong admissibility with eta = sqrt(d); N(i) = same-level
boxes that are not admissible; IL(i) = children of N(P(i)) that are not in N(i).

Readings: R1 "no more than n_max" (<=) and L >= 2; R2 bounding cube
centred at the per-axis midpoint; R3 integer box coordinates from one exact
IEEE evaluation at level LMAX, coarser levels by shift, half-open boxes with a
closed global upper face; R4 Morton order with axis 0 least significant; R5
admissibility == Chebyshev index distance >= 2 (exact for eta = sqrt(d)); R6
greedy first-fit colouring in Morton order with conflict = neighbours.
"""
from __future__ import annotations

import numpy as np

LMAX = 20          # integer coordinates are computed once at this level (R3)


def root_box(points: np.ndarray):
    """P:122 smallest hypercube containing the support (R2). Returns (g, two_h)."""
    lo = points.min(axis=0)
    hi = points.max(axis=0)
    c = (lo + hi) / 2.0
    h = np.max(hi - lo) / 2.0
    if not h > 0.0:
        h = 2.0 ** -20          # degenerate cloud (single point / all coincident)
    g = c - h                   # lower corner
    return g, 2.0 * h


def int_coords(points: np.ndarray, g: np.ndarray, two_h: float) -> np.ndarray:
    """R3: k_a = clamp(floor(((p_a - g_a) / (2h)) * 2^LMAX), 0, 2^LMAX - 1).

    numpy evaluates each elementwise op in IEEE round-to-nearest without FMA
    contraction, which the CUDA path reproduces with __dsub_rn/__ddiv_rn.
    """
    t = (points - g) / two_h
    t = t * float(1 << LMAX)
    k = np.floor(t).astype(np.int64)
    return np.clip(k, 0, (1 << LMAX) - 1)


def morton(coords: np.ndarray, bits: int) -> np.ndarray:
    """R4: interleave coordinate bits, axis 0 least significant."""
    n, d = coords.shape
    key = np.zeros(n, dtype=np.int64)
    for b in range(bits):
        for a in range(d):
            key |= ((coords[:, a] >> b) & 1) << (b * d + a)
    return key


def choose_depth(kc: np.ndarray, d: int, n_max: int) -> int:
    """R1: smallest L >= 2 with every box holding <= n_max points."""
    for L in range(2, LMAX + 1):
        lvl = kc >> (LMAX - L)
        keys = morton(lvl, L)
        _, counts = np.unique(keys, return_counts=True)
        if counts.max() <= n_max:
            return L
        if d * L > 24:
            break
    raise ValueError("cannot subdivide: coincident points or too deep a tree")


class Tree:
    """Uniform 2^d tree over sorted points.

    perm[j] = user index of the j-th point in tree order.
    off[l] : int64[2^(d l) + 1], points of box b at level l are perm[off[l][b]:off[l][b+1]].
    coords(l, b) : integer box coordinates (de-interleaved Morton id).
    """

    def __init__(self, points: np.ndarray, n_max: int):
        points = np.asarray(points, dtype=np.float64)
        n, d = points.shape
        if n < 1:
            raise ValueError("empty input")
        if d not in (2, 3):
            raise ValueError("d must be 2 or 3")
        self.d, self.n, self.n_max = d, n, n_max
        self.g, self.two_h = root_box(points)
        kc = int_coords(points, self.g, self.two_h)
        self.L = choose_depth(kc, d, n_max)
        leaf = morton(kc >> (LMAX - self.L), self.L)
        # stable sort by (leaf Morton id, original index)
        self.perm = np.lexsort((np.arange(n), leaf)).astype(np.int64)
        self.sorted_leaf_key = leaf[self.perm]
        self.points = points[self.perm]                # tree order
        self.off = {}
        for l in range(0, self.L + 1):
            lk = self.sorted_leaf_key >> (d * (self.L - l))
            self.off[l] = np.searchsorted(lk, np.arange((1 << (d * l)) + 1), side="left").astype(np.int64)

    # --- geometry helpers -------------------------------------------------
    def nboxes(self, l):
        return 1 << (self.d * l)

    def count(self, l, b):
        return int(self.off[l][b + 1] - self.off[l][b])

    def nonempty(self, l):
        o = self.off[l]
        return [b for b in range(self.nboxes(l)) if o[b + 1] > o[b]]

    def coords(self, l, b):
        c = [0] * self.d
        for bit in range(l):
            for a in range(self.d):
                c[a] |= ((b >> (bit * self.d + a)) & 1) << bit
        return tuple(c)

    def box_id(self, c, l):
        b = 0
        for bit in range(l):
            for a in range(self.d):
                b |= ((c[a] >> bit) & 1) << (bit * self.d + a)
        return b

    def point_range(self, l, b):
        return int(self.off[l][b]), int(self.off[l][b + 1])

    def children(self, l, b):
        """Non-empty children of box b at level l, Morton order."""
        out = []
        for j in range(1 << self.d):
            c = (b << self.d) | j
            if self.count(l + 1, c) > 0:
                out.append(c)
        return out


def chebyshev(t: Tree, l, a, b):
    ca, cb = t.coords(l, a), t.coords(l, b)
    return max(abs(x - y) for x, y in zip(ca, cb))


def admissible_geometric(t: Tree, l, a, b):
    """Eq. adm_condn on box geometry in units of the box side:
    max(diam) <= eta * dist, eta = sqrt(d), diam = sqrt(d), dist = Euclidean gap.
    Evaluated in exact integer arithmetic (squared): d <= d * gap^2."""
    ca, cb = t.coords(l, a), t.coords(l, b)
    gap2 = sum(max(0, abs(x - y) - 1) ** 2 for x, y in zip(ca, cb))
    return gap2 * t.d >= t.d and gap2 > 0


def build_lists(t: Tree):
    """N(i) and IL(i) per level >= 2 (Table; Remark P:402-404).

    Returns near[l][b] (sorted, includes b) and il[l][b] (sorted), for non-empty b.
    """
    near, il = {}, {}
    for l in range(2, t.L + 1):
        near[l], il[l] = {}, {}
        side = 1 << l
        ne = set(t.nonempty(l))
        for b in sorted(ne):
            c = t.coords(l, b)
            nb = []
            for off in np.ndindex(*([3] * t.d)):
                cc = tuple(c[a] + off[a] - 1 for a in range(t.d))
                if all(0 <= x < side for x in cc):
                    j = t.box_id(cc, l)
                    if j in ne:
                        nb.append(j)
            near[l][b] = sorted(nb)
            # children of the parent's neighbours that are not neighbours
            pc = tuple(x >> 1 for x in c)
            cand = []
            for off in np.ndindex(*([3] * t.d)):
                pp = tuple(pc[a] + off[a] - 1 for a in range(t.d))
                if all(0 <= x < (side >> 1) for x in pp):
                    pb = t.box_id(pp, l - 1)
                    for j in range(1 << t.d):
                        ch = (pb << t.d) | j
                        if ch in ne and max(abs(x - y) for x, y in zip(t.coords(l, ch), c)) >= 2:
                            cand.append(ch)
            il[l][b] = sorted(cand)
    return near, il


def greedy_colours(t: Tree, near_l: dict):
    """R6: greedy first-fit in Morton order; conflict = N(i) minus i."""
    col = {}
    for b in sorted(near_l):
        used = {col[j] for j in near_l[b] if j in col}
        c = 0
        while c in used:
            c += 1
        col[b] = c
    return col
