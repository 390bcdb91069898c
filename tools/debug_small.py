import sys, numpy as np
sys.path.insert(0, '.')
import paper_2007_13552_b200.api as dnd
from oracle.bind import Oracle
O = Oracle(); comm = dnd.Communicator(0)
for n in [300, 256, 512, 1000, 5000, 100_000]:
    for m in (18, 32):
        xh = O.uniform_f32(n, m, 5 + n)
        x = dnd.from_global(xh, (n, m), 0, comm)
        init = xh[:8].astype(np.float64)
        mod = dnd.kmeans_fit(x, 8, 1, 0.0, 1, init=init)
        c_ref, t_ref, _ = O.kmeans_lloyd(xh.astype(np.float64), init, 1)
        lab = O.kmeans_predict(xh.astype(np.float64), init)
        cnt = np.bincount(lab, minlength=8)
        sums = np.stack([xh[lab == j].astype(np.float64).sum(0) for j in range(8)])
        got_sums = mod.centroids * cnt[:, None]
        print(n, m, "maxdev", np.max(np.abs(mod.centroids - c_ref)), "trace", mod.inertia_trace[0], t_ref[0])
        if np.max(np.abs(mod.centroids - c_ref)) > 1e-5:
            print("  counts", cnt.tolist())
            print("  sumdiff per cluster", np.abs(got_sums - sums).max(1).round(3).tolist())
