"""Cached oracle results for the BASELINE configs too large to re-run inside a test (north_star /
BASELINE.md "CPU baseline plan": computed once, cached, keyed by config hash).

Runs ONLY the serial C++ oracle (oracle/cpp.py; OpenMP over independent boxes, bit-identical to
one thread) and the seeded input generators -- nothing from the CUDA path -- and writes
tests/golden/<workload>_oracle.npz:
  x          the oracle's solution (user order, N x nrhs)
  ranks_<l>  final box ranks after the factorization (level l, all 2^(d l) boxes)
  nnca_<l>   NNCA ranks
  residual   ||A x - b|| / ||b|| over the 4096 sampled rows (exact direct sum, oracle/dense.py)
  meta       JSON: config, config hash, times, threads, host
Usage: python tools/oracle_golden.py <config number 1-5> [threads] [n_override] [out_dir]
(out_dir defaults to tests/golden; the GPU box's host writes to gpurun_out/ and the file is
copied into tests/golden afterwards.)
"""
import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import dense                           # noqa: E402
from oracle.cpp import CppAIFMM                    # noqa: E402
from paper_2301_12704_b200 import workloads as W   # noqa: E402


def config_hash(cfg, n):
    return hashlib.sha256(json.dumps({**cfg.__dict__, "n": n}, sort_keys=True).encode()).hexdigest()[:16]


def main():
    ci = int(sys.argv[1])
    threads = int(sys.argv[2]) if len(sys.argv) > 2 else (os.cpu_count() or 1)
    cfg = W.CONFIGS[ci - 1]
    n = int(sys.argv[3]) if len(sys.argv) > 3 and int(sys.argv[3]) > 0 else cfg.n
    pts, b = W.make(cfg, n=n)
    t0 = time.time()
    o = CppAIFMM(pts, cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol, threads=threads)
    print(f"build {time.time() - t0:.1f}s L={o.L}", flush=True)
    o.factor()
    print(f"factor done {time.time() - t0:.1f}s", flush=True)
    x = o.solve(b)
    st = o.stats()
    ranks = {l: (o.ranks(l, 1), o.ranks(l, 0)) for l in range(2, o.L + 1)}
    L = o.L
    del o                                            # free the factorization before the residual
    rows = W.residual_rows(n, cfg.seed)
    res = dense.residual(pts, cfg.kernel_id, cfg.kparams, x, b, rows)
    meta = {"workload": cfg.name, "n": n, "config_hash": config_hash(cfg, n), "threads": threads,
            "host": platform.node(), "cpu": platform.processor(), "nproc": os.cpu_count(),
            "times_s": st, "residual_4096_rows": res, "L": L, "script": "tools/oracle_golden.py",
            "oracle": "oracle/cpp/aifmm_oracle.cpp (serial C++, OpenMP bit-identical)"}
    out = {"x": x, "meta": np.array(json.dumps(meta))}
    for l, (rf, rn) in ranks.items():
        out[f"ranks_{l}"] = rf
        out[f"nnca_{l}"] = rn
    tag = cfg.name if n == cfg.n else f"{cfg.name}_n{n}"
    out_dir = sys.argv[4] if len(sys.argv) > 4 else os.path.join(ROOT, "tests", "golden")
    path = os.path.join(out_dir, f"{tag}_oracle.npz")
    np.savez_compressed(path, **out)
    print(json.dumps(meta), flush=True)


if __name__ == "__main__":
    main()
