"""Measure the cuBLAS FP64 DGEMM rate on this B200 (roofline denominator for DMMA kernels).

MEASURED_PEAKS.json has no FP64 entry; this probe records one under the same
protocol (best of 10 with CUDA events, burst) plus a 4 s sustained loop.
"""
import json, time, subprocess, torch

def main():
    dev = torch.device("cuda:0")
    out = {"gpu": torch.cuda.get_device_name(0)}
    for n in (4096, 8192):
        a = torch.randn(n, n, dtype=torch.float64, device=dev)
        b = torch.randn(n, n, dtype=torch.float64, device=dev)
        for _ in range(3):
            torch.matmul(a, b)
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(10):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); torch.matmul(a, b); e.record(); torch.cuda.synchronize()
            best = min(best, s.elapsed_time(e) / 1e3)
        out[f"dgemm_{n}_tflops_burst"] = 2 * n**3 / best / 1e12
    # sustained
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cnt = 0; t0 = time.time(); s.record()
    while time.time() - t0 < 4.0:
        torch.matmul(a, b); cnt += 1
        if cnt % 4 == 0: torch.cuda.synchronize()
    e.record(); torch.cuda.synchronize()
    out["dgemm_8192_tflops_sustained"] = 2 * n**3 * cnt / (s.elapsed_time(e) / 1e3) / 1e12
    # copy bandwidth fp64
    x = torch.empty(2**28, dtype=torch.float64, device=dev); y = torch.empty_like(x)
    for _ in range(3): y.copy_(x)
    torch.cuda.synchronize(); best = 1e30
    for _ in range(10):
        s.record(); y.copy_(x); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    out["copy_gbs"] = 2 * x.numel() * 8 / best / 1e9
    out["props"] = str(torch.cuda.get_device_properties(0))
    print(json.dumps(out, indent=1))
    with open("gpurun_out/fp64_peak.json", "w") as f:
        json.dump(out, f, indent=1)

if __name__ == "__main__":
    main()
