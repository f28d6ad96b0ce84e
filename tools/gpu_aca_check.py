"""Cluster-ACA vs oracle rank parity on upper-level-heavy problems (debug aid)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2301_12704_b200 import aifmm as A, workloads as W
from oracle.factor import AIFMM
for (kind, n, d, kid, kp, leaf, tol) in [("uniform_pm1", 20000, 2, 0, (10.0, 0.0), 16, 1e-8),
                                          ("uniform_01", 12000, 3, 2, (100.0, 0.0), 32, 1e-6)]:
    pts = W.make_points(kind, n, d, 7)
    o = AIFMM(pts, kid, kp, leaf, tol)
    A.free()
    A.build(torch.from_numpy(pts).cuda(), kid, kp, leaf, tol)
    perm, L = A.get_tree(n)
    bad = 0; tot = 0
    for l in range(2, L + 1):
        r = A.get_ranks(l, d, 0)
        for b in o.near[l]:
            tot += 1
            if int(r[b]) != o.nnca.rank(l, b):
                bad += 1
    print(kind, n, "L", L, "rank mismatches", bad, "of", tot, flush=True)
