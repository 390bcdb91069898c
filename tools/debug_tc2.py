import os, sys, numpy as np
sys.path.insert(0, '.')
import paper_2007_13552_b200.api as dnd
comm = dnd.Communicator(0)
g = np.load('tests/golden/reference_golden.npz')
for n in (100_000, 1_000_000, 2_500_000, 5_000_000):
    x = dnd.random_uniform((n, 18), 0, 42, comm)
    out = {}
    for kind in ("tc", "small"):
        os.environ["DNDC_KMEANS_KERNEL"] = kind
        out[kind] = dnd.kmeans_fit(x, 8, 1, 0.0, 42)
    d = np.abs(out["tc"].centroids - out["small"].centroids).max()
    print(n, "tc vs small centroid maxdiff", d, "inertia", out["tc"].inertia_trace[0], out["small"].inertia_trace[0])
    if n == 5_000_000:
        print("vs golden it1: tc", np.abs(out["tc"].centroids - g["cfg1_centroids_it1"]).max(),
              "small", np.abs(out["small"].centroids - g["cfg1_centroids_it1"]).max())
