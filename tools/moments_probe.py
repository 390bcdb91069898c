"""Time dnd.moments_axis0 (host-synchronous API call) and its kernels for a few
widths: python tools/moments_probe.py"""
import time

import torch

import paper_2007_13552_b200.api as dnd

comm = dnd.Communicator(0)
for n, m in [(5_000_000, 18), (5_000_000, 16), (5_000_000, 20), (5_000_000, 32), (2_812_500, 32), (100_000_000, 32)]:
    a = dnd.random_uniform((n, m), 0, 42, comm)
    for _ in range(3):
        dnd.moments_axis0(a)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 20
    for _ in range(reps):
        dnd.moments_axis0(a)
    dt = (time.perf_counter() - t0) / reps
    print(f"n={n} m={m}: {dt*1e3:.3f} ms/call  {4*n*m/dt/1e9:.0f} GB/s", flush=True)
    del a
