"""A/B timing of alternative builds of libdndc.so (variants/*.so) on cfg1:
assign-kernel time and a 20-iteration fit, each in its own process."""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import ctypes as C, sys, torch, numpy as np
sys.path.insert(0, ".")
import paper_2007_13552_b200.api as dnd
from paper_2007_13552_b200 import _lib
comm = dnd.Communicator(0)
n, m, k = 5_000_000, 18, 8
x = dnd.random_uniform((n, m), 0, 42, comm)
ms, by = C.c_double(), C.c_double()
_lib.check(_lib.lib().dndc_kmeans_time_assign_f32(comm.handle, x.tile.data_ptr(), n, m, k, 50, C.byref(ms), C.byref(by)))
for _ in range(3): mod = dnd.kmeans_fit(x, k, 20, 0.0, 42)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); s.record()
for _ in range(5): mod = dnd.kmeans_fit(x, k, 20, 0.0, 42)
e.record(); torch.cuda.synchronize()
L = _lib.lib()
_lib.check(L.dndc_kmeans_assign_timing(comm.handle, 1))
mod = dnd.kmeans_fit(x, k, 20, 0.0, 42)
tot, nl = C.c_double(), C.c_int()
_lib.check(L.dndc_kmeans_last_assign_ms(comm.handle, C.byref(tot), C.byref(nl)))
per = (C.c_double * 64)()
L.dndc_internal_assign_times.restype = C.c_int
npl = L.dndc_internal_assign_times(comm.handle, per, 64)
per_s = " ".join(f"{per[i]*1e3:.0f}" for i in range(npl))
_lib.check(L.dndc_kmeans_assign_timing(comm.handle, 0))
g = np.load("tests/golden/reference_golden.npz")
rel = float(np.max(np.abs(mod.centroids - g["cfg1_centroids"]) / np.maximum(1, np.abs(g["cfg1_centroids"]))))
print("per-launch us:", per_s)
print(f"full-mode assign {ms.value*1e3:6.1f} us | in-fit assign avg {tot.value/nl.value*1e3:6.1f} us ({by.value/(tot.value/nl.value)/1e6:5.0f} GB/s) | iters/s {100/(s.elapsed_time(e)/1e3):7.0f} | rel {rel:.1e} refined {mod.refined_rows}")
'''
libs = sys.argv[1:] or sorted(glob.glob(os.path.join(ROOT, "variants", "*.so")))
for lib in libs:
    env = dict(os.environ, DNDC_LIB_PATH=lib)
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    print(f"{os.path.basename(lib):24s}", (r.stdout.strip() or r.stderr.strip()[-400:]), flush=True)
