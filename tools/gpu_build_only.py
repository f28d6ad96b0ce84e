"""Build (tree + lists + NNCA) timing and NNCA-rank check against the cached C++-oracle golden.
Usage: python tools/gpu_build_only.py <config index>"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2301_12704_b200 import aifmm as A, workloads as W
cfg = W.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
pts, _ = W.make(cfg)
P = torch.from_numpy(pts).cuda()
gp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", f"{cfg.name}_oracle.npz")
g = np.load(gp) if os.path.exists(gp) else None
ts = []
for rep in range(3):
    A.free(); torch.cuda.synchronize(); t0 = time.time()
    A.build(P, cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol); torch.cuda.synchronize(); ts.append(time.time() - t0)
_, L = A.get_tree(cfg.n)
ok = None if g is None else all(np.array_equal(A.get_ranks(l, cfg.d, 0), g[f"nnca_{l}"]) for l in range(2, L + 1))
print(json.dumps({"cfg": cfg.name, "build_s": ts, "nnca_ranks_equal_golden": ok, "env": os.environ.get("AIFMM_ACA_CLUSTER_NF")}), flush=True)
