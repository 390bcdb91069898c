"""Measured dense TF32 tensor-core peak of this B200 (the cfg4 roofline denominator).

    python tools/tf32_peak.py [--out profiles/tf32_peak.json]

MEASURED_PEAKS.json (driver-written) holds the copy bandwidth and the bf16
GEMM peak but no TF32 figure.  This measures it the same way the driver
measures bf16: cuBLAS fp32 GEMM with TF32 math (torch.backends.cuda.matmul.
allow_tf32) at 8192^3, 2*N^3 flops per call, CUDA events, best of 10 (burst)
and back to back for ~4 s (sustained), with NVML clocks sampled meanwhile.
The 3xTF32 cdist issues three TF32 MMAs per useful product, so its ceiling in
useful fp32 FLOP/s is tf32_peak / 3.
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/tf32_peak.json")
    ap.add_argument("--n", type=int, default=8192)
    args = ap.parse_args()
    import torch

    from bench import ClockSampler

    torch.backends.cuda.matmul.allow_tf32 = True
    torch.backends.cuda.matmul.fp32_precision = "tf32" if hasattr(torch.backends.cuda.matmul, "fp32_precision") else None
    n = args.n
    a = torch.rand(n, n, device="cuda")
    b = torch.rand(n, n, device="cuda")
    c = torch.empty(n, n, device="cuda")
    flops = 2.0 * n ** 3
    for _ in range(5):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    burst = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        e1.synchronize()
        burst.append(flops / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    clk = ClockSampler(torch.cuda.current_device())
    clk.start()
    t_end = time.time() + 4.0
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    reps = 0
    e0.record()
    while time.time() < t_end:
        for _ in range(20):
            torch.matmul(a, b, out=c)
        reps += 20
        torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    clocks = clk.stop()
    sustained = flops * reps / (e0.elapsed_time(e1) * 1e-3) / 1e12
    # fp32 without TF32 (CUDA-core FFMA) for context
    torch.backends.cuda.matmul.allow_tf32 = False
    if hasattr(torch.backends.cuda.matmul, "fp32_precision"):
        torch.backends.cuda.matmul.fp32_precision = "ieee"
    torch.matmul(a, b, out=c)
    e0.record()
    torch.matmul(a, b, out=c)
    e1.record()
    e1.synchronize()
    fp32 = flops / (e0.elapsed_time(e1) * 1e-3) / 1e12
    out = {"tf32_tflops": max(burst), "tf32_tflops_sustained": sustained,
           "tf32_burst_median": statistics.median(burst), "fp32_ffma_tflops": fp32,
           "n": n, "how": "cuBLAS fp32 GEMM with allow_tf32, 2*N^3 flops, CUDA events; best of 10 (burst) and "
                          "back to back for 4 s (sustained)",
           "clocks_sustained": clocks, "gpu": torch.cuda.get_device_name()}
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    json.dump(out, open(args.out, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
