"""Work split of the §8(e) subtree partition, measured with `world` in-process ranks on one GPU
(tests/test_gpu_dist.py's transport): per rank, the FLOPs it executed in the split phases
(Schur updates, pivot inverses, RRQR stage 1) and the bytes it received in exchanges, next to
the single-rank totals; the ranks' solutions must be bitwise identical.  Device times of ranks
sharing one GPU are not scaling numbers, so none are reported; the output is the load balance
(max over ranks / (total / world)) and the exchange volume that a multi-GPU run would see.
Run with AIFMM_DIST_FORCE=1 so that the single-rank baseline takes the distributed code path
(R31 off) too.  Usage: AIFMM_DIST_FORCE=1 python tools/gpu_dist_scaling.py <config index> [n]"""
import json
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2301_12704_b200 import aifmm as G, workloads as W

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
cfg = W.CONFIGS[ci]
pts, b = W.make(cfg, n=n)
N = pts.shape[0]
KEYS = ("schur_flops", "pivot_flops", "tri_flops", "mult_flops", "dist_bytes", "dist_exchanges", "compressions")
libs = {}


def run(world):
    shared = G.local_shared()
    out, errs = {}, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            if r not in libs:
                libs[r] = G.load_copy(r)
            with torch.cuda.stream(s), G.use(libs[r]):
                G.free()
                G.reset_counters()
                G.dist_init_local(r, world, shared, -1)   # world 1 too (AIFMM_DIST_FORCE=1: same path)
                G.build(torch.from_numpy(pts).cuda(), cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol)
                G.factor()
                x = G.solve(torch.from_numpy(np.ascontiguousarray(b)).cuda()).cpu().numpy()
                st = G.stats()
                out[r] = (x, {k: st[k] for k in KEYS})
                G.dist_finalize()
                G.free()
                s.synchronize()
        except Exception as e:  # noqa: BLE001
            errs.append((r, repr(e)))

    th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(world)]
    [t.start() for t in th]
    [t.join(1800) for t in th]
    assert not errs, errs
    return out


base = run(1)[0][1]
for world in (2, 4, 8):
    out = run(world)
    same = all(np.array_equal(out[0][0], out[r][0]) for r in range(world))
    line = {"workload": cfg.name, "n": N, "world": world, "replicas_bitwise_identical": same}
    for k in ("schur_flops", "pivot_flops", "tri_flops", "mult_flops"):
        per = [out[r][1][k] for r in range(world)]
        line[k] = {"single_rank_total": base[k], "sum_over_ranks": sum(per), "max_rank": max(per),
                   "imbalance": max(per) / (base[k] / world) if base[k] else None}
    line["exchange_gb_received_per_rank"] = [round(out[r][1]["dist_bytes"] / 1e9, 4) for r in range(world)]
    line["exchanges_per_factor"] = out[0][1]["dist_exchanges"]
    print(json.dumps(line), flush=True)
