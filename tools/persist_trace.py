"""Timeline of the persistent k-means fit (cfg1) from %globaltimer marks.

    DNDC_PERSIST_TRACE=1 python tools/persist_trace.py [--rows 5000000] [--iters 20]

Per iteration: time from CTA 0's start to its update, the spread of the CTAs'
tiles-done times (first / median / last), the barrier release after the last
CTA, and the update.  Diagnostics only.
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=5_000_000)
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    os.environ.setdefault("DNDC_PERSIST_TRACE", "1")
    import torch

    import paper_2007_13552_b200.api as dnd
    from paper_2007_13552_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world > 1:  # under torchrun: one rank per GPU, rank 0 prints its own timeline
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        comm = dnd.Communicator.from_torch_distributed(local)
    else:
        comm = dnd.Communicator(0)
    x = dnd.random_uniform((args.rows, 18), 0, 42, comm)
    for _ in range(3):
        dnd.kmeans_fit(x, 8, args.iters, 0.0, 42)
    L = _lib.lib()
    L.dndc_kmeans_persist_trace.restype = C.c_int64
    cap = args.iters * (2 * 4096 + 2)
    buf = np.zeros(cap, np.uint64)
    grid = C.c_int()
    n = L.dndc_kmeans_persist_trace(comm.handle, buf.ctypes.data_as(C.c_void_p), C.c_int64(cap), C.byref(grid))
    G = grid.value
    if n == 0:
        print("no trace (DNDC_PERSIST_TRACE unset or not the persistent kernel)")
        return
    if int(os.environ.get("RANK", 0)) != 0:
        return
    m = buf[:n].reshape(args.iters, 2 * G + 2).astype(np.int64)
    t0 = m[0, 2 * G]
    print(f"trace stride {G} CTAs (grids may differ per launch; unused slots are 0); times in us")
    print("iter    start   tiles: first   median     last  released  upd_done  iter_us")
    for it in range(args.iters):
        st = (m[it, 2 * G] - t0) / 1e3
        td_raw, rel_raw = m[it, :G], m[it, G:2 * G]
        td = (td_raw[td_raw > 0] - t0) / 1e3
        rel = (rel_raw[rel_raw > 0] - t0) / 1e3
        up = (m[it, 2 * G + 1] - t0) / 1e3
        print(f"{it:4d} {st:8.1f}  {td.min():8.1f} {np.median(td):8.1f} {td.max():8.1f}  {rel.max():8.1f}  "
              f"{up:8.1f}  {up - st:7.1f}")
    print(f"total {(m[-1, 2 * G + 1] - t0) / 1e3:.1f} us")


if __name__ == "__main__":
    main()
