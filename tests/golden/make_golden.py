"""Generates tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run here, where /root/reference exists:  python tests/golden/make_golden.py
The fixtures are small and committed; the GPU box never needs the reference.
Inputs are the reference's own synthetic data, random_uniform<float>
(ndarray.hpp:154-169), widened exactly to f64 as the parity contract states
(BASELINE.md section 4).
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.bind import Reference  # noqa: E402


def main() -> None:
    R = Reference()
    out = {}

    # A1: generator samples (row blocks of the cfg1 and cfg5 arrays)
    x = R.uniform_f32(4096, 18, 42, p=3)
    out["uniform_18_s42_head"] = x
    out["uniform_32_s7_head"] = R.uniform_f32(1024, 32, 7, p=2)

    # A2: chunk maps
    for n, p in [(5, 3), (3, 5), (5_000_000, 8), (200_000, 3), (100_000_000, 8)]:
        off, ext = R.chunk_map(n, p)
        out[f"chunk_{n}_{p}"] = np.stack([off, ext])

    # A3-A7: cdist on 300 x 18 (p = 1, 3) and cdist_xy vs a 37-row y
    a = R.uniform_f32(300, 18, 71, p=1).astype(np.float64)
    out["cdist_x"] = a
    out["cdist_p1"], _ = R.cdist(a, 1)
    d3, sr = R.cdist(a, 3)
    out["cdist_p3"] = d3
    out["cdist_p3_sendrecvs"] = np.array([sr])
    y = R.uniform_f32(37, 18, 43, p=1).astype(np.float64)
    out["cdist_y"] = y
    out["cdist_xy"] = R.cdist_xy(a, y, 2)
    out["row_norms_x"] = R.row_norms(a)

    # A11: init indices
    for n, k, s in [(100, 8, 21), (6, 6, 77), (5_000_000, 8, 42), (100_000_000, 8, 42), (50_000_000, 64, 42)]:
        out[f"init_{n}_{k}_{s}"] = R.kmeans_init_indices(n, k, s)

    # A8-A12: k-means 600 x 8, k = 8, 30 iterations at p = 1, 2, 4
    km = R.uniform_f32(600, 8, 109, p=1).astype(np.float64)
    out["km600_x"] = km
    for p in (1, 2, 4):
        c, t, it = R.kmeans_fit(km, 8, 30, 0.0, 42, p)
        out[f"km600_p{p}_centroids"] = c
        out[f"km600_p{p}_trace"] = t
    out["km600_labels"] = R.kmeans_predict(km, out["km600_p1_centroids"], 1)
    # tol > 0 stops early (cluster.cpp:149-150)
    c, t, it = R.kmeans_fit(km, 8, 100, 1e-3, 42, 3)
    out["km600_tol_centroids"], out["km600_tol_trace"], out["km600_tol_iters"] = c, t, np.array([it])

    # cfg1 at full size: 5M x 18, k = 8, 20 Lloyd iterations, seed 42 (8 ranks)
    c, t, it = R.kmeans_fit_synthetic(5_000_000, 18, 42, 8, 20, 0.0, 42, p=8)
    out["cfg1_centroids"], out["cfg1_trace"] = c, t
    # cfg1 trajectory: the centroids after t iterations (kmeans_fit is
    # deterministic, so max_iter = t reproduces iteration t's state)
    for t_it in (1, 5):
        c, t, it = R.kmeans_fit_synthetic(5_000_000, 18, 42, 8, t_it, 0.0, 42, p=8)
        out[f"cfg1_centroids_it{t_it}"] = c

    # A13/A14: moments along split axis 0
    mo = R.uniform_f32(1000, 18, 59, p=1).astype(np.float64)
    out["mom_x"] = mo
    for p in (1, 3, 5):
        mean, var = R.moments_axis0(mo, p, 0)
        out[f"mom_p{p}_mean"], out[f"mom_p{p}_var"] = mean, var
    mean, var = R.moments_axis0(mo, 2, 1)
    out["mom_p2_ddof1_var"] = var

    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print(f"wrote {len(out)} arrays")


if __name__ == "__main__":
    main()
