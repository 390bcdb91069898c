"""Per-tile event times of kmeans_tcd_kernel on CTA 0 (needs a -DTCD_TRACE build:
make -C paper_2007_13552_b200/csrc EXTRA=-DTCD_TRACE).  cfg3 shard fit, then
the marks of the last tcd launch, in us from the first hi issue."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_13552_b200.api as dnd  # noqa: E402
from paper_2007_13552_b200 import _lib  # noqa: E402

comm = dnd.Communicator(0)
x = dnd.random_uniform((6_250_000, 64), 0, 42, comm)
dnd.kmeans_fit(x, 64, 4, 0.0, 42)
buf = np.zeros(512, np.uint64)
L = _lib.lib()
L.dndc_internal_tcd_trace.argtypes = [ctypes.c_void_p]
_lib.check(L.dndc_internal_tcd_trace(buf.ctypes.data))
m = buf.reshape(64, 8).astype(np.float64)
t0 = m[0, 0]
names = ["hi", "lo", "full", "hidone", "lodone", "dfull", "dempty", "end"]
print("tile " + " ".join(f"{n:>8s}" for n in names))
for i in range(64):
    print(f"{i:4d} " + " ".join(f"{(v - t0) / 1e3:8.2f}" if v else "       -" for v in m[i]))
