"""Summarise an `ncu --set full` capture of one kernel (read with `ncu -i REP --page raw --csv`):
per-launch duration, DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum), FP64 tensor-pipe
(DMMA) utilisation, achieved occupancy, top stall reasons.  Writes a JSON summary (bench.py reads
the DRAM bytes per launch for roofline.traffic).

Usage: python tools/ncu_kernel_traffic.py REP.ncu-rep OUT.json [kernel-regex]"""
import csv
import io
import json
import re
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
pat = re.compile(sys.argv[3] if len(sys.argv) > 3 else ".")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, data = rows[0], rows[1], [r for r in rows[2:] if pat.search(r[rows[0].index("Kernel Name")])]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0,
         "ms": 1e3, "msecond": 1e3}


def _f(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return float("nan")


def col(name):
    """values of one metric over the captured launches; launches where ncu could not collect
    it (n/a, e.g. a launch replayed in fewer passes) are dropped"""
    if name not in h:
        return None
    i = h.index(name)
    v = [_f(r[i]) * SCALE.get(units[i], 1.0) for r in data]
    v = [x for x in v if x == x]
    return v or None


def mean(v):
    return sum(v) / len(v) if v else None


dur = col("gpu__time_duration.sum")                       # us
rd, wr = col("dram__bytes_read.sum"), col("dram__bytes_write.sum")
dmma = col("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active")
occ = col("sm__warps_active.avg.pct_of_peak_sustained_active")
stalls = {}
for i, k in enumerate(h):
    m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio", k)
    if m:
        v = [x for x in (_f(r[i]) for r in data) if x == x]
        if v:
            stalls[m.group(1)] = sum(v) / len(v)
n = len(data)
summary = {
    "report": rep, "kernel_filter": pat.pattern, "launches_captured": n,
    "launches_with_dram_metrics": len(rd) if rd else 0,
    "kernel": data[0][h.index("Kernel Name")].split("(")[0] if n else None,
    "mean_duration_us": mean(dur),
    "dram_bytes_per_launch": (mean(rd) + mean(wr)) if rd and wr else None,
    "dram_read_bytes_per_launch": mean(rd),
    "dram_write_bytes_per_launch": mean(wr),
    "dmma_pipe_pct_of_peak_active": mean(dmma),
    "warps_active_pct": mean(occ),
    "top_stalls_per_issue": dict(sorted(stalls.items(), key=lambda x: -x[1])[:6]),
    "note": "ncu --set full --clock-control none: cold caches, serialised launches (absolute times "
            "are not bench values)",
}
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps(summary, indent=1))
