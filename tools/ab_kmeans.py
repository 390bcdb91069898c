"""A/B timing of the k-means assign kernels (tc / small / generic) + cfg1 parity."""
import ctypes as C, os, sys, numpy as np
sys.path.insert(0, '.')
import paper_2007_13552_b200.api as dnd
from paper_2007_13552_b200 import _lib
comm = dnd.Communicator(0)
g = np.load('tests/golden/reference_golden.npz')
def rel(a, b): return float(np.max(np.abs(a - b) / np.maximum(1, np.abs(b))))
shapes = [(5_000_000, 18, 8)] + ([(6_250_000, 64, 64)] if "cfg3" in sys.argv else [])
for (n, m, k) in shapes:
    x = dnd.random_uniform((n, m), 0, 42, comm)
    for kind in ("tc", "small", "generic"):
        if kind == "small" and m != 18: continue
        os.environ["DNDC_KMEANS_KERNEL"] = kind
        ms, by = C.c_double(), C.c_double()
        _lib.check(_lib.lib().dndc_kmeans_time_assign_f32(comm.handle, x.tile.data_ptr(), n, m, k, 20, C.byref(ms), C.byref(by)))
        line = f"{n}x{m} k={k} {kind:8s} assign {ms.value*1e3:8.1f} us  {by.value/ms.value/1e6:7.0f} GB/s"
        if m == 18:
            mod = dnd.kmeans_fit(x, k, 20, 0.0, 42)
            line += f"  it20 rel {rel(mod.centroids, g['cfg1_centroids']):.2e} refined {mod.refined_rows}"
        print(line, flush=True)
