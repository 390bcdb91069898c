"""BASELINE config 4 for ncu: cdist_xy(100k x 1024, 100k x 1024) through the
tcgen05 3xTF32 kernel (one warm call, then the profiled one)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_13552_b200.api as dnd  # noqa: E402
from paper_2007_13552_b200 import _lib  # noqa: E402

comm = dnd.Communicator(0)
n, m = 100_000, 1024
x = dnd.random_uniform((n, m), 0, 42, comm)
y = dnd.random_uniform((n, m), 0, 43, comm)
out = torch.empty((n, n), dtype=torch.float32, device="cuda")
L = _lib.lib()
for _ in range(2):
    _lib.check(L.dndc_cdist_xy_ring_f32(comm.handle, x.tile.data_ptr(), n, y.tile.data_ptr(), n, n, m, out.data_ptr()))
torch.cuda.synchronize()
print("cfg4 ok", float(out[0, :4].sum()))
