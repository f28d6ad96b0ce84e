"""bench.py — AIFMM factor+solve throughput on B200 (BASELINE.json metric).

Workload (N=1): BASELINE config 3, the largest configuration that fits one GPU — 2D,
N = 1,048,576 uniform random points in [-1,1]^2 (seed 2), Matern-1/2 A_ij = exp(-|x_i-x_j|/0.1)
with A_ii = 1 + 1e-2, leaf 128, tol 1e-8, 1 RHS.  One step = the whole hot path (SURVEY §8(a)
rows a1-a7): aifmm_build (tree, lists, colours, NNCA), aifmm_factor (colour-batched Alg. 3)
and aifmm_solve (Alg. 4).  Inputs are resident in HBM when the timed region starts; L2
(126 MB) is flushed by writing a 256 MB buffer between steps (the step's working set is
~160 GB anyway).  `--cfg 2` selects BASELINE config 2 (N = 65,536, log r, 16 RHS).

N>1 (torchrun): the SAME workload factored by all ranks together:
the tree is split by subtrees at a coarse level, each rank compresses, inverts and updates the
blocks of its own subtrees and the ranks exchange the results over NCCL after every phase
(aifmm_dist_init); strong scaling, value = N / (max over ranks of factor + solve time).

--impl reference: the serial C++ oracle (oracle/cpp, one thread) on a bounded sample of the same
workload (the first 16384 points of the same draw), timed on the host (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2301_12704_b200 import workloads as W  # noqa: E402
from paper_2301_12704_b200 import dist as D  # noqa: E402

METRIC = "AIFMM factor+solve unknowns/sec"
UNIT = "unknowns/s"
CFG_DEFAULT = 3               # BASELINE config 3: the largest single-GPU configuration
SAMPLE_N = {2: 16384, 3: 16384}  # oracle sample size (same distribution, kernel, leaf, tol, nrhs)
KERNEL_NAMES = {0: "log r", 1: "exp(-r/ell)", 2: "1/r"}


def _peaks():
    out = {"hbm_gbs": None, "bf16_tflops": None}
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        out.update(hbm_gbs=mp.get("hbm_gbs"), bf16_tflops=mp.get("bf16_tflops"))
    except Exception:
        pass
    try:
        fp = json.load(open(os.path.join(ROOT, "profiles", "r01_fp64_dgemm_peak.json")))
        out["fp64_dgemm_tflops"] = fp.get("dgemm_8192_tflops_burst")
    except Exception:
        out["fp64_dgemm_tflops"] = None
    return out


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region (profiling recipe)."""

    def __init__(self, index=0):
        self.index, self.samples, self.proc = index, [], None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm = [float(s[0]) for s in self.samples if len(s) >= 7 and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) >= 7 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            if len(s) < 7:
                continue
            for nm, v in zip(names, s[3:7]):
                if v.strip().lower() in ("active", "1"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


ORACLE_THREADS = 1            # the north_star's "plain serial CPU C++" oracle: one core


def _oracle_sample(cfg, n):
    """The serial C++ oracle (oracle/cpp, plain loops, one thread) on a bounded sample: the
    first `n` points of a draw with the config's distribution and seed (same kernel, diagonal,
    leaf size, tol, nrhs).  Times from the oracle's own steady_clock per phase."""
    from oracle.cpp import CppAIFMM
    pts, b = W.make(cfg, n=n)
    o = CppAIFMM(pts, cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol, threads=ORACLE_THREADS)
    o.factor()
    o.solve(b)
    st = o.stats()
    return {"build_s": st["build_s"], "factor_s": st["factor_s"], "solve_s": st["solve_s"], "n": n}


def _cores():
    return ORACLE_THREADS


def _host():
    try:
        model = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name"))
    except Exception:
        model = "?"
    return f"{model}, {os.cpu_count()} logical CPUs on the host"


def _config_dict(cfg, **extra):
    d = {"workload": cfg.name, "n": cfg.n, "nrhs": cfg.nrhs,
         "kernel": f"{KERNEL_NAMES[cfg.kernel_id]}, A_ii={cfg.diag:g}" + (f", ell={cfg.ell:g}" if cfg.kernel_id == 1 else ""),
         "leaf": cfg.leaf_size, "tol": cfg.tol}
    d.update(extra)
    return d


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # bounded per-step sample: the cpu_baseline sample, halved when many steps are requested so
    # that the whole --steps K run stays within a few minutes (~8 s per 8192-point step)
    sn = SAMPLE_N[args.cfg] if args.steps <= 5 else SAMPLE_N[args.cfg] // 2
    times = []
    for _ in range(args.warmup):          # warm up on a tiny instance
        _oracle_sample(cfg, 1024)
    for _ in range(max(1, args.steps)):
        r = _oracle_sample(cfg, sn)
        times.append(r)
    fs = [t["factor_s"] + t["solve_s"] for t in times]
    value = sn / float(np.mean(fs))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": len(times), "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean([t["build_s"] + t["factor_s"] + t["solve_s"] for t in times])),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config_dict(cfg, sample_n=sn),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": _cores(), "kind": "oracle",
                         "sample": f"serial C++ oracle (oracle/cpp) on the first {sn} points of the {cfg.name} draw "
                                   f"(seed {cfg.seed}), same kernel/leaf/tol/{cfg.nrhs} RHS; host: {_host()}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "phase_s": {k: float(np.mean([t[k] for t in times])) for k in ("build_s", "factor_s", "solve_s")},
    }
    print(json.dumps(line), flush=True)


def _phase_roofline(name, kernels, bound, work, ms, peak, unit, launches=None):
    achieved = (work / (ms / 1e3)) / (1e12 if unit == "TFLOP/s" else 1e9) if ms > 0 else None
    return {"phase": name, "kernels": kernels, "bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
            "frac": (achieved / peak) if (achieved and peak) else None, "device_ms_per_step": ms,
            ("algorithmic_tflop_per_step" if unit == "TFLOP/s" else "algorithmic_gb_per_step"):
                work / (1e12 if unit == "TFLOP/s" else 1e9)}


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist
    from paper_2301_12704_b200 import aifmm as A

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    A.load()
    A.set_stream(stream.cuda_stream)

    # N > 1: all ranks factor the same workload together (subtree split, NCCL exchanges inside
    # the library): rank 0 creates the library's NCCL id, the others receive it
    if world > 1:
        A.dist_init(rank, world, D.share_unique_id(A.dist_unique_id() if rank == 0 else None))
    cfg_r = cfg
    pts, b = W.make(cfg_r)
    P = torch.from_numpy(pts).to(dev)
    B = torch.from_numpy(np.ascontiguousarray(b)).to(dev)
    Bcm = B.t().contiguous()                                  # column-major n x nrhs
    flush = torch.empty(256 << 20 >> 3, dtype=torch.float64, device=dev)

    def step(timing=False):
        A.free()
        A.set_timing(timing)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        X = Bcm.clone()
        e[0].record(stream)
        A.build(P, cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol)
        e[1].record(stream)
        A.factor()
        e[2].record(stream)
        A.solve_device_ptr(X.data_ptr(), cfg.nrhs)
        e[3].record(stream)
        return e, X

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    A.reset_counters()
    tb = tf = ts = 0.0
    acc = {}
    launches = 0.0
    keys = ("schur_ms", "schur_flops", "schur_bytes", "schur_launches", "pivot_ms", "pivot_flops", "pivot_bytes",
            "tri_ms", "tri_flops", "tri_bytes", "pqr_ms", "pqr_bytes", "redir_ms", "redir_flops", "redir_bytes",
            "factor_flops", "max_rank", "compressions", "device_bytes", "host_syncs", "dist_bytes", "dist_exchanges",
            "mult_ms", "mult_flops", "proj_ms", "proj_flops", "fresh_ms", "fresh_flops", "orth_ms")
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        e, X = step(timing=True)
        torch.cuda.synchronize()
        tb += e[0].elapsed_time(e[1])
        tf += e[1].elapsed_time(e[2])
        ts += e[2].elapsed_time(e[3])
        st = A.stats()
        for k in keys:
            acc[k] = acc.get(k, 0.0) + st[k]
        launches += st["launches"]
        A.reset_counters()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    K = float(args.steps)
    step_ms = (tb + tf + ts) / K
    fs_ms = (tf + ts) / K
    fs_ms, step_ms = D.max_over_ranks([fs_ms, step_ms], dev)
    value = D.strong_throughput(cfg.n, fs_ms / 1e3)

    # correctness guard on the last device result: direct-sum residual on the GPU (row a9,
    # aifmm_residual) over the 4096 sampled rows
    Xu = X.t()
    res = A.residual(Xu, B, W.residual_rows(cfg.n, cfg_r.seed))

    # end-to-end: host points + host B through the public API, copies inside the region
    # (one untimed warm-up, then the mean of up to 3 timed runs)
    pts_h = torch.from_numpy(pts).pin_memory()
    Bh = np.asfortranarray(b.copy())
    torch.cuda.synchronize()
    e2e_t = []
    for it in range(1 + max(1, min(args.steps, 3))):
        A.free()
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        Pd = pts_h.to(dev, non_blocking=True)
        A.build(Pd, cfg.kernel_id, cfg.kparams, cfg.leaf_size, cfg.tol)
        A.factor()
        Xh = A.solve_host(Bh.copy())
        torch.cuda.synchronize()
        if it > 0:
            e2e_t.append(time.perf_counter() - t0)
    e2e_value = D.strong_throughput(cfg.n, D.max_over_ranks([float(np.mean(e2e_t))], dev)[0])

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    pk = _peaks()
    fp64 = pk.get("fp64_dgemm_tflops") or (pk["bf16_tflops"] * 45.0 / 2250.0 if pk["bf16_tflops"] else None)
    hbm = pk.get("hbm_gbs")
    # DRAM traffic per Schur launch from the committed `ncu --set full` capture of exactly these
    # launches (NVTX range "schur"; tools/ncu_kernel_traffic.py), next to the algorithmic bytes
    traffic, ncu_src = None, None
    try:
        nc = json.load(open(os.path.join(ROOT, "profiles", f"r02_schur_gemm_ncu_cfg{args.cfg}.json")))
        traffic, ncu_src = nc.get("dram_bytes_per_launch"), nc
    except Exception:
        pass
    sch_ms = acc["schur_ms"] / K
    achieved = (acc["schur_flops"] / K) / (sch_ms / 1e3) / 1e12 if sch_ms > 0 else None
    roof = {
        "kernel": "gemm_tasks_kernel (Schur-complement updates, DMMA)",
        "bound": "tensor", "achieved": achieved, "peak": fp64, "unit": "TFLOP/s",
        "frac": (achieved / fp64) if (achieved and fp64) else None,
        "traffic": traffic,
        "traffic_source": (f"profiles/r02_schur_gemm_ncu_cfg{args.cfg}.json: mean dram__bytes_read.sum + "
                           f"dram__bytes_write.sum over {ncu_src['launches_captured']} captured Schur launches") if ncu_src else None,
        "algorithmic_bytes_per_launch": (acc["schur_bytes"] / acc["schur_launches"]) if acc["schur_launches"] else None,
        "algorithmic_flop_per_launch": (acc["schur_flops"] / acc["schur_launches"]) if acc["schur_launches"] else None,
        "launches_per_step": acc["schur_launches"] / K,
        "peak_source": "FP64 (DMMA) peak = cuBLAS DGEMM 8192^3 measured on this pool "
                       "(profiles/r01_fp64_dgemm_peak.json); MEASURED_PEAKS.json has no FP64 entry",
        "schur_ms_per_step": sch_ms, "schur_gflop_per_step": acc["schur_flops"] / K / 1e9,
    }
    phases = [
        _phase_roofline("pivot factorisation (P_i^-1, P:753)", "gj_small_kernel / gj_panel_* + DMMA GEMM", "tensor",
                        acc["pivot_flops"] / K, acc["pivot_ms"] / K, fp64, "TFLOP/s"),
        _phase_roofline("RRQR stage 1 (Householder of W^T, R8b; 2 n m^2 flops, DMMA trailing updates)",
                        "hh_panel_* + hh_update_kernel", "tensor", acc["tri_flops"] / K, acc["tri_ms"] / K, fp64, "TFLOP/s"),
        _phase_roofline("RRQR stage 2 (truncated pivoted QR, P:841-849)", "pqr_tasks_kernel / pqr_cluster_kernel", "hbm",
                        acc["pqr_bytes"] / K, acc["pqr_ms"] / K, hbm, "GB/s"),
        _phase_roofline("redirection (P:877-882, P:1010-1014, P:1078-1082)", "gemm_tasks_kernel", "hbm",
                        acc["redir_bytes"] / K, acc["redir_ms"] / K, hbm, "GB/s"),
        _phase_roofline("multipliers W_i = G_i[:, :m] R_i (P:753)", "gemm_tasks_kernel", "tensor",
                        acc["mult_flops"] / K, acc["mult_ms"] / K, fp64, "TFLOP/s"),
        _phase_roofline("compression projections (I - U U^T) F (P:841-849, R8)", "gemm_tasks_kernel", "tensor",
                        acc["proj_flops"] / K, acc["proj_ms"] / K, fp64, "TFLOP/s"),
        _phase_roofline("new blocks C_p G12, G21 R_q, -G22 (Table 4 P:649-677)", "gemm_tasks_kernel + copy_tasks_kernel",
                        "tensor", acc["fresh_flops"] / K, acc["fresh_ms"] / K, fp64, "TFLOP/s"),
    ]
    phase_ms = {k: acc[k + "_ms"] / K for k in ("schur", "pivot", "tri", "pqr", "redir", "mult", "proj", "fresh", "orth")}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        sn = SAMPLE_N[args.cfg]
        r = _oracle_sample(cfg, sn)
        cpu = {"value": sn / (r["factor_s"] + r["solve_s"]), "unit": UNIT, "cores": _cores(), "kind": "oracle",
               "sample": f"serial C++ oracle (oracle/cpp) on the first {sn} points of the {cfg.name} draw (seed {cfg.seed}), "
                         f"same kernel/leaf/tol/{cfg.nrhs} RHS; build {r['build_s']:.1f}s factor {r['factor_s']:.1f}s "
                         f"solve {r['solve_s']:.1f}s; host: {_host()}"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config_dict(cfg, parallelism="1 GPU" if world == 1 else
                               f"{world} GPUs: subtree split, owner computes, NCCL broadcast exchanges per phase",
                               l2="flushed (256 MB write) between steps; working set > L2"),
        "phase_ms": {"build": tb / K, "factor": tf / K, "solve": ts / K},
        "factor_phase_device_ms": phase_ms,
        "rel_residual_4096_rows": res,
        "factor_tflop_per_step": acc["factor_flops"] / K / 1e12,
        "max_rank": acc["max_rank"] / K, "compressions_per_step": acc["compressions"] / K,
        "device_gb": acc["device_bytes"] / K / 1e9, "host_syncs_per_step": acc["host_syncs"] / K,
        "dist_exchange_gb_per_step": acc["dist_bytes"] / K / 1e9, "dist_exchanges_per_step": acc["dist_exchanges"] / K,
        "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_step": [round(t * 1e3, 2) for t in e2e_t],
                "h2d_bytes_per_step": int(pts.nbytes + b.nbytes),
                "d2h_bytes_per_step": int(b.nbytes), "includes": "H2D points, build, factor, H2D B, solve, D2H X; warm-up run excluded"},
        "gpu_launches": int(launches / K),
        "roofline": roof,
        "roofline_phases": phases,
        "cpu_baseline": cpu,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cfg", type=int, default=CFG_DEFAULT, choices=[2, 3], help="BASELINE config number")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    cfg = W.CONFIGS[args.cfg - 1]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
