import os, sys, numpy as np
sys.path.insert(0, '.')
import paper_2007_13552_b200.api as dnd
from oracle.bind import Oracle
O = Oracle(); comm = dnd.Communicator(0)
g = np.load('tests/golden/reference_golden.npz')
n, m = 2_000_000, 18
x = dnd.random_uniform((n, m), 0, 42, comm)
xh = x.tile.cpu().numpy().astype(np.float64)
for key in ("cfg1_centroids_it1", "cfg1_centroids_it5", "cfg1_centroids"):
    cents = g[key]
    model = dnd.KMeansModel(8, 18, cents)
    res = {}
    for kind in ("tc", "small"):
        os.environ["DNDC_KMEANS_KERNEL"] = kind
        res[kind] = dnd.gather(dnd.kmeans_predict(model, x))
        res[kind + "_ref"] = model.refined_rows
    ref = O.kmeans_predict(xh, cents)
    for kind in ("tc", "small"):
        bad = np.nonzero(res[kind] != ref)[0]
        print(key, kind, "mismatches", len(bad))
        if len(bad):
            d2 = ((xh[bad[:5], None, :] - cents[None]) ** 2).sum(-1)
            srt = np.sort(d2, 1)
            print("   gaps of first mismatches", (srt[:, 1] - srt[:, 0]).tolist())
