"""Two in-process ranks on a small case with AIFMM_DEBUG_DIST=1 (per-phase state digests)."""
import os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2301_12704_b200 import aifmm as G, workloads as W

world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 6000
pts = W.make_points("uniform_pm1", n, 2, 60)
nrhs = int(sys.argv[3]) if len(sys.argv) > 3 else 1
b = W.make_rhs(n, nrhs, 60)
shared = G.local_shared()
libs = [G.load_copy(r) for r in range(world)]
out = {}
def body(r):
    torch.cuda.set_device(0)
    s = torch.cuda.Stream() if (len(sys.argv) <= 4 or sys.argv[4] != "nostream") else torch.cuda.default_stream()
    with torch.cuda.stream(s), G.use(libs[r]):
        G.free()
        G.set_algorithm(3)
        G.dist_init_local(r, world, shared, -1)
        G.build(torch.from_numpy(pts).cuda(), 0, (10.0, 0.0), 32, 1e-8)
        G.factor()
        out[r] = G.solve(torch.from_numpy(np.ascontiguousarray(b)).cuda()).cpu().numpy()
        out[r] = (out[r], G.solve(torch.from_numpy(np.ascontiguousarray(b[:, :1])).cuda()).cpu().numpy())
th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(world)]
[t.start() for t in th]
[t.join(300) for t in th]
print("equal:", all(np.array_equal(out[0][0], out[r][0]) for r in range(world)),
      "1-col equal:", all(np.array_equal(out[0][1], out[r][1]) for r in range(world)),
      "norms", [float(np.linalg.norm(out[r][0])) for r in range(world)], [float(np.linalg.norm(out[r][1])) for r in range(world)], flush=True)
