"""Config-5 preconditioner quality from the serial C++ oracle alone (no CUDA path): for the
config-5 distribution (3D uniform [0,1)^3, 1/r, A_ii = 100, leaf 128) at reduced N, the AIFMM
factorization at eps_A = 1e-3 (BASELINE) and 1e-5 (the paper's Exp. 5 value) applied
to b ~ N(0,1): relative residual ||A M^-1 b - b|| / ||b|| by exact direct sum on 4096 sampled
rows.  A value >= 1 means M^-1 is no preconditioner at that N.
Usage: python tools/oracle_cfg5_precond.py [threads] N1 N2 ...  -> one JSON line per (N, eps)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import dense                           # noqa: E402
from oracle.cpp import CppAIFMM                    # noqa: E402
from paper_2301_12704_b200 import workloads as W   # noqa: E402

cfg = W.CONFIGS[4]
threads = int(sys.argv[1])
for n in [int(a) for a in sys.argv[2:]]:
    pts, b = W.make(cfg, n=n)
    rows = W.residual_rows(n, cfg.seed)
    for eps in (1e-3, 1e-5):
        t0 = time.time()
        o = CppAIFMM(pts, cfg.kernel_id, cfg.kparams, cfg.leaf_size, eps, threads=threads).factor()
        x = o.solve(b)
        st = o.stats()
        del o
        r = dense.residual(pts, cfg.kernel_id, cfg.kparams, x, b, rows)
        print(json.dumps({"n": n, "eps": eps, "precond_rel_residual": r, "build_s": st["build_s"],
                          "factor_s": st["factor_s"], "wall_s": time.time() - t0, "threads": threads}), flush=True)
