"""Config-2 full-size decision parity: oracle once, GPU variants (env toggles) vs it."""
import os, sys, json, subprocess
sys.path.insert(0, '.')
import numpy as np
if len(sys.argv) > 1 and sys.argv[1] == "gpu":
    import torch
    from paper_2301_12704_b200 import aifmm as G, workloads as W
    from oracle import dense
    cfg = W.CONFIGS[1]
    pts, b = W.make(cfg)
    G.build(torch.from_numpy(pts).cuda(), cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol)
    G.factor()
    x = G.solve(torch.from_numpy(np.ascontiguousarray(b)).cuda()).cpu().numpy()
    perm, L = G.get_tree(cfg.n)
    ranks = {l: G.get_ranks(l, 2, 1).tolist() for l in range(2, L + 1)}
    np.save("/tmp/x_gpu.npy", x)
    json.dump(ranks, open("/tmp/ranks_gpu.json", "w"))
    sys.exit(0)
from paper_2301_12704_b200 import workloads as W
from oracle.factor import AIFMM as Oracle
cfg = W.CONFIGS[1]
pts, b = W.make(cfg)
o = Oracle(pts, cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol).factor()
xo = o.solve(b)
for name, env in [("default", {}), ("orth_pqr", {"AIFMM_ORTH_PQR": "1"}), ("hh_cluster", {"AIFMM_HH_CLUSTER": "1"}),
                  ("both_old", {"AIFMM_ORTH_PQR": "1", "AIFMM_HH_CLUSTER": "1"})]:
    e = dict(os.environ); e.update(env)
    subprocess.run([sys.executable, __file__, "gpu"], env=e, check=True)
    x = np.load("/tmp/x_gpu.npy"); rk = json.load(open("/tmp/ranks_gpu.json"))
    mism = {l: sum(1 for bx in o.levels[int(l)].boxes if rk[l][bx] != o.levels[int(l)].k[bx]) for l in rk}
    print(name, "rel", float(np.linalg.norm(x - xo) / np.linalg.norm(xo)), "rank mismatches", mism, flush=True)
