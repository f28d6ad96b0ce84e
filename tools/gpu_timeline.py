"""GPU timeline of one config-2 factor (torch.profiler / CUPTI sees the library's kernels too):
GPU-busy time vs wall time, per-kernel totals (real clocks, concurrent, warm caches) and the
largest idle gaps.  Usage: python tools/gpu_timeline.py [cfg_index] [n]"""
import json
import sys
import time

sys.path.insert(0, '.')
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2301_12704_b200 import aifmm as A, workloads as W

cfgi = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
cfg = W.CONFIGS[cfgi]
pts, b = W.make(cfg, n=n)
P = torch.from_numpy(pts).cuda()
B = torch.from_numpy(np.ascontiguousarray(b)).cuda()


def step():
    A.free()
    A.build(P, cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    A.factor()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    A.solve(B)
    torch.cuda.synchronize()
    return t0, t1


for _ in range(2):
    step()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0, t1 = step()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ks = sorted([(e.time_range.start, e.time_range.end, e.name) for e in evs], key=lambda x: x[0])
# restrict to the factor window: kernels between the first and last aifmm kernel after build
# (use the wall-clock split: factor = t1 - t0; align by the biggest gap heuristic is fragile,
# so report the whole step and the factor wall time separately)
busy = 0.0
cur_s = cur_e = None
gaps = []
prev_nm = ''
for s, e, nm in ks:
    if cur_e is not None and e > cur_e:
        pass
    if cur_e is None:
        cur_s, cur_e = s, e
        continue
    if s > cur_e:
        busy += cur_e - cur_s
        gaps.append((s - cur_e, prev_nm.split('(')[0][:40] + ' -> ' + nm.split('(')[0][:40]))
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
    prev_nm = nm
if cur_e is not None:
    busy += cur_e - cur_s
span = ks[-1][1] - ks[0][0] if ks else 0
tot = {}
for s, e, nm in ks:
    k = nm.split('(')[0].replace('void ', '')[:60]
    a = tot.setdefault(k, [0.0, 0])
    a[0] += e - s
    a[1] += 1
print(json.dumps({"cfg": cfg.name, "n": len(pts), "factor_wall_ms": (t1 - t0) * 1e3,
                  "kernels": len(ks), "gpu_span_ms": span / 1e3, "gpu_busy_ms": busy / 1e3,
                  "idle_ms": (span - busy) / 1e3}))
for k, (t, c) in sorted(tot.items(), key=lambda x: -x[1][0])[:30]:
    print(f"{t / 1e3:10.2f} ms {c:6d}  {k}")
gaps.sort(key=lambda x: -x[0])
print("largest idle gaps (us, next kernel):")
for g, nm in gaps[:40]:
    print(f"{g:10.1f}  {nm[:90]}")
hist = [0, 0, 0, 0, 0]
hsum = [0.0] * 5
for g, _ in gaps:
    i = 0 if g < 10 else 1 if g < 50 else 2 if g < 200 else 3 if g < 1000 else 4
    hist[i] += 1
    hsum[i] += g
print("gap histogram <10us, <50, <200, <1000, >=1000:", hist, [round(x / 1e3, 2) for x in hsum], "ms")
