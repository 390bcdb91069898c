import os, sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
import paper_2007_13552_b200.api as dnd
from oracle.bind import Oracle
O = Oracle()
os.environ["DNDC_KMEANS_KERNEL"] = "tc"
comm = dnd.Communicator(0)
n, m, k = 2048, 64, 64
xh = O.uniform_f32(n, m, 11)
x = dnd.from_global(xh, (n, m), 0, comm)
c_ref, t_ref, _ = O.kmeans_fit(xh.astype(np.float64), k, 6, 0.0, 3)
for it in range(1, 7):
    mdl = dnd.kmeans_fit(x, k, it, 0.0, 3)
    print(it, "trace", np.array(mdl.inertia_trace) - np.array(t_ref[:it]))
    c_i, _, _ = O.kmeans_fit(xh.astype(np.float64), k, it, 0.0, 3)
    print("  cent dev", np.max(np.abs(mdl.centroids - c_i)))
