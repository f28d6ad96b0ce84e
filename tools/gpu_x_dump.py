"""Config-2 GPU solution written to gpurun_out/x_<tag>.npy (for GPU-vs-GPU / GPU-vs-oracle
rounding comparisons made on the CPU side)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2301_12704_b200 import aifmm as A, workloads as W
tag = sys.argv[1]
cfg = W.CONFIGS[1]
pts, b = W.make(cfg)
A.build(torch.from_numpy(pts).cuda(), cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol)
A.factor()
x = A.solve(torch.from_numpy(np.ascontiguousarray(b)).cuda()).cpu().numpy()
np.save(f"gpurun_out/x_{tag}.npy", x)
print(tag, "done")
