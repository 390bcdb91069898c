"""Config-size golden fixtures from the UNMODIFIED reference (oracle/_ref).

    python tests/golden/make_golden_cfg.py      (here, where /root/reference exists)

Writes tests/golden/cfg_golden.npz (a few tens of KB):
  * cfg1 (5M x 18, k=8, 20 iterations, 8 ranks): the reference's labels for its
    own final centroids (kmeans_predict, cluster.cpp:155-172) as per-cluster
    counts plus an order-sensitive digest (tests/_parity.py:label_digest);
  * cfg3 slice (5M x 64, k=64, 20 iterations, 8 ranks):
    centroids, inertia trace, counts and label digest.
The 50M-row cfg3 needs ~100 GB of host f64 for the reference; the 5M slice is
the survey's stated parity case.  Takes a few minutes on 8 cores.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from oracle.bind import Reference  # noqa: E402
from _parity import label_digest  # noqa: E402


def main() -> None:
    R = Reference()
    old = np.load(os.path.join(HERE, "reference_golden.npz"))
    out = {}
    t0 = time.time()
    # cfg1: labels of the reference's 20-iteration centroids
    x = R.uniform_f32(5_000_000, 18, 42, p=8).astype(np.float64)
    lab = R.kmeans_predict(x, old["cfg1_centroids"], 8)
    out["cfg1_counts"] = np.bincount(lab, minlength=8).astype(np.int64)
    out["cfg1_label_digest"] = np.array([label_digest(lab)], np.uint64)
    del x, lab
    print(f"cfg1 labels {time.time() - t0:.0f} s", flush=True)
    # cfg3 slice: 5M x 64, k = 64
    for it in (1, 20):
        c, t, n_it = R.kmeans_fit_synthetic(5_000_000, 64, 42, 64, it, 0.0, 42, p=8)
        out[f"cfg3s_centroids_it{it}"] = c
        out[f"cfg3s_trace_it{it}"] = t
        print(f"cfg3 slice {it} iterations {time.time() - t0:.0f} s", flush=True)
    x = R.uniform_f32(5_000_000, 64, 42, p=8).astype(np.float64)
    lab = R.kmeans_predict(x, out["cfg3s_centroids_it20"], 8)
    out["cfg3s_counts"] = np.bincount(lab, minlength=64).astype(np.int64)
    out["cfg3s_label_digest"] = np.array([label_digest(lab)], np.uint64)
    np.savez_compressed(os.path.join(HERE, "cfg_golden.npz"), **out)
    print(f"wrote {len(out)} arrays in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
