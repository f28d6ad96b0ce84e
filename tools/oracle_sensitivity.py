"""Rounding sensitivity of the oracle itself on BASELINE config 2 (full size), written to
tests/golden/cfg2_oracle_rounding_sensitivity.json.  Calls only oracle/ and the seeded input
generators (no CUDA path).

Two runs of the oracle that differ only in HOW the pivot inverse P_i^{-1} (reading R16) is
rounded: numpy.linalg.inv (LAPACK getrf + getri) vs an LU solve against the identity
(getrf + getrs).  Both are exact in exact arithmetic; their relative 2-norm solution difference
is the method's own sensitivity to the rounding of one step -- the floor below which no
implementation (GPU or CPU) can be compared with the oracle (reading R24)."""
import json
import os
import sys
import time

import numpy as np
import scipy.linalg as sl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle.factor as F                         # noqa: E402
from paper_2301_12704_b200 import workloads as W  # noqa: E402


def main():
    cfg = W.CONFIGS[1]
    pts, b = W.make(cfg)
    t0 = time.time()
    o1 = F.AIFMM(pts, cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol).factor()
    x1 = o1.solve(b)
    inv = F.np.linalg.inv

    def inv_lu(P):
        return sl.lu_solve(sl.lu_factor(P), np.eye(P.shape[0]))

    F.np.linalg.inv = inv_lu
    try:
        o2 = F.AIFMM(pts, cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol).factor()
        x2 = o2.solve(b)
    finally:
        F.np.linalg.inv = inv
    rel = float(np.linalg.norm(x2 - x1) / np.linalg.norm(x1))
    mism = {str(l): int(sum(1 for bx in o1.levels[l].boxes if o1.levels[l].k[bx] != o2.levels[l].k[bx]))
            for l in o1.levels}
    out = {"workload": cfg.name, "tol": cfg.tol,
           "rel_solution_diff_inv_vs_lu_solve": rel,
           "final_rank_mismatches_per_level": mism,
           "seconds": time.time() - t0,
           "script": "tools/oracle_sensitivity.py"}
    path = os.path.join(ROOT, "tests", "golden", "cfg2_oracle_rounding_sensitivity.json")
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
