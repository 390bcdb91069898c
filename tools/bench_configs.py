"""Timings of BASELINE configs 2-5 on one GPU (CUDA events, device-resident inputs).

    python tools/bench_configs.py [cfg2] [cfg4] [cfg5] [cfg3]

Prints one JSON object per config with the algorithmic bytes / flops of SURVEY.md
section 8(d) and the achieved rate.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_13552_b200.api as dnd  # noqa: E402

PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json"))).get("hbm_gbs", 6538.9)


def timed(fn, reps=3, warm=1):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps / 1e3


def main():
    want = set(sys.argv[1:]) or {"cfg2", "cfg4", "cfg5", "cfg3"}
    comm = dnd.Communicator(0)
    if "cfg2" in want:
        n, m = 200_000, 18
        x = dnd.random_uniform((n, m), 0, 42, comm)
        y = dnd.random_uniform((n, m), 0, 43, comm)
        yr = dnd.DndArray((n, m), None, comm, y.tile)
        out = torch.empty((n, n), dtype=torch.float32, device="cuda")
        from paper_2007_13552_b200 import _lib
        L = _lib.lib()

        def run():
            _lib.check(L.dndc_cdist_xy_f32(comm.handle, x.tile.data_ptr(), n, y.tile.data_ptr(), n, m, out.data_ptr()))

        t = timed(run)
        byt = 4.0 * n * n + 4.0 * 2 * n * m
        print(json.dumps({"config": "cfg2 cdist_xy 200k x 18 vs 200k x 18 (1 GPU)", "seconds": t,
                          "GB/s": byt / t / 1e9, "frac_hbm": byt / t / 1e9 / PEAK,
                          "pairs_per_s": n * n / t, "TFLOP/s": 2.0 * n * n * m / t / 1e12}), flush=True)

        # self mode cdist(X) (pairwise.cpp:37-85), reported separately
        def run_self():
            _lib.check(L.dndc_cdist_f32(comm.handle, x.tile.data_ptr(), n, n, m, out.data_ptr()))

        t = timed(run_self)
        byt = 4.0 * n * n + 4.0 * n * m
        print(json.dumps({"config": "cfg2 self cdist(X) 200k x 18 (1 GPU, diagonal zeroed)", "seconds": t,
                          "GB/s": byt / t / 1e9, "frac_hbm": byt / t / 1e9 / PEAK,
                          "pairs_per_s": n * n / t}), flush=True)
        del out
        torch.cuda.empty_cache()
    if "cfg4" in want:
        n, m = 100_000, 1024
        x = dnd.random_uniform((n, m), 0, 42, comm)
        y = dnd.random_uniform((n, m), 0, 43, comm)
        out = torch.empty((n, n), dtype=torch.float32, device="cuda")
        from paper_2007_13552_b200 import _lib
        L = _lib.lib()

        def run():
            _lib.check(L.dndc_cdist_xy_f32(comm.handle, x.tile.data_ptr(), n, y.tile.data_ptr(), n, m, out.data_ptr()))

        t = timed(run, reps=1, warm=1)
        print(json.dumps({"config": "cfg4 cdist_xy 100k x 1024 vs 100k x 1024 (1 GPU)", "seconds": t,
                          "TFLOP/s": 2.0 * n * n * m / t / 1e12, "GB/s_out": 4.0 * n * n / t / 1e9}), flush=True)
        del out
        torch.cuda.empty_cache()
    if "cfg5" in want:
        n, m = 100_000_000, 32
        x = dnd.random_uniform((n, m), 0, 42, comm)
        t = timed(lambda: dnd.moments_axis0(x))
        byt = 4.0 * n * m
        print(json.dumps({"config": "cfg5 moments 100M x 32 (1 GPU, mean+M2 in one pass)", "seconds": t,
                          "GB/s": byt / t / 1e9, "frac_hbm": byt / t / 1e9 / PEAK}), flush=True)
        t = timed(lambda: dnd.kmeanspp_indices(x, 8, 42), reps=1)
        byt = 7 * (4.0 * n * m + 16.0 * n)
        print(json.dumps({"config": "cfg5 k-means++ k=8 on 100M x 32 (1 GPU)", "seconds": t,
                          "GB/s": byt / t / 1e9, "frac_hbm": byt / t / 1e9 / PEAK}), flush=True)
        del x
        torch.cuda.empty_cache()
    if "cfg3" in want:
        n, m, k = 6_250_000, 64, 64  # one GPU's shard of 50M x 64 at p = 8
        x = dnd.random_uniform((n, m), 0, 42, comm)
        t = timed(lambda: dnd.kmeans_fit(x, k, 20, 0.0, 42), reps=1)
        byt = 4.0 * n * m * 20
        print(json.dumps({"config": "cfg3 k-means k=64 20 iters on a 6.25M x 64 shard (1 GPU = 1/8 of 50M)",
                          "seconds": t, "iters_per_s": 20 / t, "GB/s": byt / t / 1e9,
                          "frac_hbm": byt / t / 1e9 / PEAK}), flush=True)


if __name__ == "__main__":
    main()
