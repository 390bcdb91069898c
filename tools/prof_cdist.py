"""ncu driver: one cdist_xy tile launch (n x n x m)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2007_13552_b200.api as dnd
from paper_2007_13552_b200 import _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 18
comm = dnd.Communicator(0)
x = dnd.random_uniform((n, m), 0, 42, comm)
y = dnd.random_uniform((n, m), 0, 43, comm)
out = torch.empty((n, n), dtype=torch.float32, device="cuda")
for _ in range(2):
    _lib.check(_lib.lib().dndc_cdist_xy_f32(comm.handle, x.tile.data_ptr(), n, y.tile.data_ptr(), n, m, out.data_ptr()))
torch.cuda.synchronize()
print("ok", float(out[1, 2]))
