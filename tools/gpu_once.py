"""One build+factor+solve of a config (for ncu launch lists)."""
import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2301_12704_b200 import aifmm as A, workloads as W
cfg = W.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
pts, b = W.make(cfg)
P = torch.from_numpy(pts).cuda(); B = torch.from_numpy(np.ascontiguousarray(b)).cuda()
A.build(P, cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol); A.factor(); X = A.solve(B)
torch.cuda.synchronize(); print("done", A.stats()["launches"])
