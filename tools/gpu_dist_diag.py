"""Config-2 solutions of: single GPU (default env), and the in-process split with `world` ranks;
saved to gpurun_out/x_<tag>.npy for comparison.  Usage: python tools/gpu_dist_diag.py tag world"""
import os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2301_12704_b200 import aifmm as G, workloads as W
tag, world = sys.argv[1], int(sys.argv[2])
cfg = W.CONFIGS[1]
pts, b = W.make(cfg)
if world == 0:
    G.build(torch.from_numpy(pts).cuda(), cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol); G.factor()
    x = G.solve(torch.from_numpy(np.ascontiguousarray(b)).cuda()).cpu().numpy()
    ranks = {l: G.get_ranks(l, 2, 1) for l in range(2, 7)}
else:
    shared = G.local_shared(); libs = [G.load_copy(r) for r in range(world)]; out = {}
    def body(r):
        torch.cuda.set_device(0); s = torch.cuda.Stream()
        with torch.cuda.stream(s), G.use(libs[r]):
            G.dist_init_local(r, world, shared, -1)
            G.build(torch.from_numpy(pts).cuda(), cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol); G.factor()
            out[r] = (G.solve(torch.from_numpy(np.ascontiguousarray(b)).cuda()).cpu().numpy(), {l: G.get_ranks(l, 2, 1) for l in range(2, 7)})
    th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(world)]
    [t.start() for t in th]; [t.join(900) for t in th]
    x, ranks = out[0]
np.save(f"gpurun_out/x_{tag}.npy", x)
np.savez(f"gpurun_out/ranks_{tag}.npz", **{str(k): v for k, v in ranks.items()})
print(tag, "done", float(np.linalg.norm(x)))
