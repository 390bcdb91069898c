"""Quick functional check of the tcgen05 k-means kernel on one shape (n m k)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_13552_b200.api as dnd  # noqa: E402
from oracle.bind import Oracle  # noqa: E402

O = Oracle()
comm = dnd.Communicator(0)
os.environ["DNDC_KMEANS_KERNEL"] = "tc"
n, m, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
xh = O.uniform_f32(n, m, 5)
x = dnd.from_global(xh, (n, m), 0, comm)
cents = O.uniform_f64(k, m, 7)
model = dnd.KMeansModel(k, m, cents)
lab = dnd.gather(dnd.kmeans_predict(model, x))
print("predict mismatches", int((lab != O.kmeans_predict(xh.astype(np.float64), cents)).sum()), flush=True)
mod = dnd.kmeans_fit(x, k, 3, 0.0, 1)
c_ref, t_ref, _ = O.kmeans_fit(xh.astype(np.float64), k, 3, 0.0, 1)
print("fit dev", float(np.max(np.abs(mod.centroids - c_ref))), "refined", mod.refined_rows, flush=True)
