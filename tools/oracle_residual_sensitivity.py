"""Rounding sensitivity of the oracle's RESIDUAL on BASELINE config 2 (full size), written to
tests/golden/cfg2_oracle_residual_sensitivity.json.  Calls only oracle/ and the seeded input
generators (no CUDA path).

Three runs of the oracle that differ only in how the pivot inverse P_i^{-1} (reading R16) is
rounded -- numpy.linalg.inv (getrf + getri), an LU solve against the identity (getrf + getrs),
and the transpose of the inverse of P_i^T -- all exact in exact arithmetic.  The spread of their
sampled direct-sum residuals (4096 rows, the rows the tests and bench.py use) is the method's
own sensitivity to the rounding of one step (reading R26)."""
import json
import os
import sys
import time

import numpy as np
import scipy.linalg as sl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle.factor as F                         # noqa: E402
from oracle import dense                          # noqa: E402
from paper_2301_12704_b200 import workloads as W  # noqa: E402


def main():
    cfg = W.CONFIGS[1]
    pts, b = W.make(cfg)
    rows = W.residual_rows(cfg.n, cfg.seed)
    inv = F.np.linalg.inv
    variants = {
        "inv": inv,
        "lu_solve": lambda P: sl.lu_solve(sl.lu_factor(P), np.eye(P.shape[0])),
        "inv_of_transpose": lambda P: inv(np.ascontiguousarray(P.T)).T,
    }
    out = {"workload": cfg.name, "tol": cfg.tol, "residual_rows": len(rows), "residuals": {}}
    t0 = time.time()
    for name, fn in variants.items():
        F.np.linalg.inv = fn
        try:
            o = F.AIFMM(pts, cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol).factor()
            x = o.solve(b)
        finally:
            F.np.linalg.inv = inv
        out["residuals"][name] = float(dense.residual(pts, cfg.kernel_id, cfg.kparams, x, b, rows))
        print(name, out["residuals"][name], flush=True)
    r = list(out["residuals"].values())
    out["max_over_min"] = max(r) / min(r)
    out["seconds"] = time.time() - t0
    out["script"] = "tools/oracle_residual_sensitivity.py"
    with open(os.path.join(ROOT, "tests", "golden", "cfg2_oracle_residual_sensitivity.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
