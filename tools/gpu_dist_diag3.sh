#!/bin/bash
AIFMM_DEBUG_DIST=2 AIFMM_DIST_FORCE=1 python tools/gpu_dist_diag.py w1 1 2> gpurun_out/dig_w1.log
AIFMM_DEBUG_DIST=2 AIFMM_DIST_PHASES=1 python tools/gpu_dist_diag.py w2_cmp 2 2> gpurun_out/dig_w2.log
python - <<'PY'
import re
def load(f):
    out = {}
    for l in open(f):
        m = re.match(r"\[dist 0\] box L4 colour 1 compressed: b=(\d+) m=(\d+) k=(\d+) own=(-?\d+) \|U\|\^2=(\S+) dev_from_unit=(\S+)", l.strip())
        if m: out[int(m.group(1))] = (int(m.group(3)), int(m.group(4)), float(m.group(5)), float(m.group(6)))
    return out
a, b = load("gpurun_out/dig_w1.log"), load("gpurun_out/dig_w2.log")
n = 0
for bx in sorted(a):
    if a[bx] != b.get(bx):
        n += 1
        if n <= 12: print(bx, "w1", a[bx], "w2", b.get(bx))
print("boxes differing:", n, "of", len(a))
PY
