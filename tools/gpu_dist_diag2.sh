#!/bin/bash
AIFMM_DEBUG_DIST=1 AIFMM_DIST_FORCE=1 python tools/gpu_dist_diag.py w1 1 2> gpurun_out/dig_w1.log
AIFMM_DEBUG_DIST=1 AIFMM_DIST_PHASES=1 python tools/gpu_dist_diag.py w2_cmp 2 2> gpurun_out/dig_w2.log
python - <<'PY'
import re
def load(f, rank):
    out = []
    for l in open(f):
        m = re.match(r"\[dist (\d+)\] (.*)", l.strip())
        if m and int(m.group(1)) == rank: out.append(m.group(2))
    return out
a, b = load("gpurun_out/dig_w1.log", 0), load("gpurun_out/dig_w2.log", 0)
print(len(a), len(b))
for x, y in zip(a, b):
    if x != y:
        print("FIRST DIFF\n w1:", x, "\n w2:", y); break
else:
    print("no diff")
PY
