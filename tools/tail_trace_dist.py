"""Fused-tail timeline per rank (torchrun; library built with -DKS_TAIL_TRACE)."""
import ctypes as C
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_13552_b200.api as dnd  # noqa: E402
from paper_2007_13552_b200 import _lib  # noqa: E402

local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
rank = dist.get_rank()
comm = dnd.Communicator.from_torch_distributed(local)
x = dnd.random_uniform((5_000_000, 18), 0, 42, comm)
L = _lib.lib()
for it in (2, 20):
    dnd.kmeans_fit(x, 8, it, 0.0, 42)
    torch.cuda.synchronize()
    t = (C.c_ulonglong * 16)()
    _lib.check(L.dndc_internal_tail_trace(t))
    b = t[5]
    line = (f"rank {rank} fit {it:2d}: last CTA {(t[1]-b)/1e3:6.1f} | reduced {(t[2]-b)/1e3:6.1f} | "
            f"exchanged {(t[3]-b)/1e3:6.1f} | updated {(t[4]-b)/1e3:6.1f} us [fold {(t[6]-t[3])/1e3:.1f} elem "
            f"{(t[7]-t[6])/1e3:.1f} clusters {(t[8]-t[7])/1e3:.1f} final {(t[4]-t[8])/1e3:.1f}]")
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, line)
    if rank == 0:
        print("\n".join(out), flush=True)
_lib.check(L.dndc_kmeans_assign_timing(comm.handle, 1))
dnd.kmeans_fit(x, 8, 20, 0.0, 42)
per = (C.c_double * 64)()
L.dndc_internal_assign_times.restype = C.c_int
n = L.dndc_internal_assign_times(comm.handle, per, 64)
line = f"rank {rank} per-launch us: " + " ".join(f"{per[i]*1e3:.0f}" for i in range(n))
out = [None] * dist.get_world_size()
dist.all_gather_object(out, line)
if rank == 0:
    print("\n".join(out), flush=True)
dist.destroy_process_group()
