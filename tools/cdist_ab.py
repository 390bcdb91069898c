"""A/B timing of cdist variants on BASELINE config 2 (200k x 18 vs 200k x 18,
one GPU): the default build and any variants/*.so given on the command line
(e.g. variants/STOREONLY.so: the same kernel writing constants, no MMA wait /
TMEM reads -- the store path's ceiling).  Each library in its own process."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, torch
sys.path.insert(0, ".")
import paper_2007_13552_b200.api as dnd
from paper_2007_13552_b200 import _lib
comm = dnd.Communicator(0)
n, m = 200_000, 18
x = dnd.random_uniform((n, m), 0, 42, comm)
y = dnd.random_uniform((n, m), 0, 43, comm)
out = torch.empty((n, n), dtype=torch.float32, device="cuda")
L = _lib.lib()
def call():
    _lib.check(L.dndc_cdist_xy_ring_f32(comm.handle, x.tile.data_ptr(), n, y.tile.data_ptr(), n, n, m, out.data_ptr()))
call(); torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(3): call()
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 3
print(f"{ms:7.2f} ms  {(4.0*n*n + 8.0*n*m)/(ms*1e-3)/1e9:7.0f} GB/s")
'''
for lib in [os.path.join(ROOT, "paper_2007_13552_b200", "libdndc.so")] + sys.argv[1:]:
    env = dict(os.environ, DNDC_LIB_PATH=lib)
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    print(f"{os.path.basename(lib):24s}", (r.stdout.strip() or r.stderr.strip()[-400:]), flush=True)
