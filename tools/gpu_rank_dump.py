"""Config-2 final ranks per level (GPU) -> gpurun_out/ranks_<tag>.npz (rank-decision comparisons)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2301_12704_b200 import aifmm as A, workloads as W
tag = sys.argv[1]
cfg = W.CONFIGS[1]
pts, b = W.make(cfg)
A.build(torch.from_numpy(pts).cuda(), cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol)
A.factor()
perm, L = A.get_tree(len(pts))
np.savez(f"gpurun_out/ranks_{tag}.npz", **{str(l): A.get_ranks(l, 2, 1) for l in range(2, L + 1)}, **{"nnca" + str(l): A.get_ranks(l, 2, 0) for l in range(2, L + 1)})
print("ok")
