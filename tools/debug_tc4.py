import os, sys, numpy as np
sys.path.insert(0, '.')
import paper_2007_13552_b200.api as dnd
from oracle.bind import Oracle
O = Oracle(); comm = dnd.Communicator(0)
x = dnd.random_uniform((5_000_000, 18), 0, 42, comm)
xh = x.tile.cpu().numpy().astype(np.float64)
os.environ["DNDC_KMEANS_KERNEL"] = "tc"
for it in (7, 8, 9):
    os.environ["DNDC_KMEANS_KERNEL"] = "tc"
    m = dnd.kmeans_fit(x, 8, it, 0.0, 42)
    labs = {}
    for kind in ("tc", "small"):
        os.environ["DNDC_KMEANS_KERNEL"] = kind
        labs[kind] = dnd.gather(dnd.kmeans_predict(m, x))
    ref = O.kmeans_predict(xh, m.centroids)
    for kind in ("tc", "small"):
        bad = np.nonzero(labs[kind] != ref)[0]
        print(it, kind, "mismatches vs oracle", len(bad), bad[:5].tolist())
        for i in bad[:3]:
            d2 = ((xh[i][None, :] - m.centroids) ** 2).sum(-1)
            o = np.argsort(d2)
            print("    row", i, "best", o[:2].tolist(), "gap", d2[o[1]] - d2[o[0]], "labels tc/small/ref", labs["tc"][i], labs["small"][i], ref[i])
