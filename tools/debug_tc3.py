import os, sys, numpy as np
sys.path.insert(0, '.')
import paper_2007_13552_b200.api as dnd
from oracle.bind import Reference
comm = dnd.Communicator(0)
g = np.load('tests/golden/reference_golden.npz')
x = dnd.random_uniform((5_000_000, 18), 0, 42, comm)
def rel(a, b): return float(np.max(np.abs(a - b) / np.maximum(1, np.abs(b))))
for kind in ("small", "tc"):
    os.environ["DNDC_KMEANS_KERNEL"] = kind
    m = dnd.kmeans_fit(x, 8, 20, 0.0, 42)
    print(kind, "it20 rel", rel(m.centroids, g["cfg1_centroids"]), "trace rel", rel(np.array(m.inertia_trace), g["cfg1_trace"]), "refined", m.refined_rows)
    tr = np.array(m.inertia_trace); gt = g["cfg1_trace"]
    print("   per-iter trace rel", [f"{v:.1e}" for v in np.abs(tr - gt) / gt])
