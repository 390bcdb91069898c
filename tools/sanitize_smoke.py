"""Small shapes of every hand-written kernel, for compute-sanitizer.

    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
    compute-sanitizer --tool synccheck python tools/sanitize_smoke.py

Persistent k-means (full + delta launches, static and dynamic tiles, ragged
last tile), the per-iteration k-means kernels, the tcgen05 k-means and cdist
paths (3xTF32, TMA, TMEM), the FFMA cdist tiles, moments, k-means++, resplit and
LASSO.  Prints one line and exits 0 when every result also matches the oracle.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_13552_b200.api as dnd  # noqa: E402
from oracle.bind import Oracle  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b)))) if a.size else 0.0


def main():
    O = Oracle()
    comm = dnd.Communicator(0)
    ok = True
    for n, m, k, it in [(70_001, 18, 8, 6), (2_000, 18, 8, 3), (5_003, 32, 8, 4), (3_000, 64, 64, 3), (999, 5, 3, 4)]:
        xh = O.uniform_f32(n, m, 7)
        x = dnd.from_global(xh, (n, m), 0, comm)
        mod = dnd.kmeans_fit(x, k, it, 0.0, 3)
        c, t, _ = O.kmeans_fit(xh.astype(np.float64), k, it, 0.0, 3)
        ok &= rel(mod.centroids, c) <= 1e-6
        lab = dnd.gather(dnd.kmeans_predict(mod, x))
        ok &= bool(np.array_equal(lab, O.kmeans_predict(xh.astype(np.float64), mod.centroids)))
    for n, ny, m in [(300, 257, 18), (200, 300, 300), (129, 131, 7)]:
        xh, yh = O.uniform_f32(n, m, 1), O.uniform_f32(ny, m, 2)
        x = dnd.from_global(xh, (n, m), 0, comm)
        y = dnd.from_global(yh, (ny, m), None, comm)
        ok &= rel(dnd.gather(dnd.cdist_xy(x, y)), O.cdist_xy(xh.astype(np.float64), yh.astype(np.float64))) <= 1e-5
        ok &= rel(dnd.gather(dnd.cdist(x)), O.cdist(xh.astype(np.float64))) <= 1e-5
    xh = O.uniform_f32(10_001, 32, 3)
    x = dnd.from_global(xh, xh.shape, 0, comm)
    st = dnd.moments_axis0(x)
    mean, var = O.moments_axis0(xh.astype(np.float64))
    ok &= rel(st.mean, mean) <= 1e-12 and rel(st.m2 / xh.shape[0], var) <= 1e-12
    ok &= bool(np.array_equal(dnd.kmeanspp_indices(x, 5, 9), O.kmeanspp_indices(xh, 5, 9)))
    r = dnd.resplit(dnd.from_global(np.arange(60.0), (5, 4, 3), 0, comm), 1)
    ok &= bool(np.array_equal(dnd.gather(r).ravel(), np.arange(60.0)))
    rng = np.random.default_rng(5)
    xl = np.hstack([np.ones((501, 1)), rng.normal(size=(501, 6))])
    yl = xl @ rng.normal(size=7)
    ml = dnd.lasso_fit(dnd.from_global(xl, xl.shape, 0, comm), dnd.from_global(yl, yl.shape, 0, comm), 0.5, 10)
    wl, _, _ = O.lasso_fit(xl, yl, 0.5, 10)
    ok &= rel(ml.weights, wl) <= 1e-9
    print("sanitize smoke", "ok" if ok else "MISMATCH")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
