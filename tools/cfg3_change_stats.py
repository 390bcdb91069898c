"""Rows whose label changes per iteration of the cfg3 shard fit (6.25M x 64,
k=64): labels after fits of 1, 2, ... iterations, compared pairwise."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_13552_b200.api as dnd  # noqa: E402

comm = dnd.Communicator(0)
x = dnd.random_uniform((6_250_000, 64), 0, 42, comm)
prev = None
pref = 0
for it in range(1, 12):
    m = dnd.kmeans_fit(x, 64, it, 0.0, 42)
    lab = dnd.gather(dnd.kmeans_predict(m, x))
    ch = None if prev is None else int(np.sum(lab != prev))
    print(f"after {it:2d} iterations: labels changed vs previous {ch}, refined {m.refined_rows - pref}", flush=True)
    prev = lab
    pref = m.refined_rows
