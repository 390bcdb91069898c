"""Timeline of the fused k-means tail (variants built with -DKS_TAIL_TRACE)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_13552_b200.api as dnd  # noqa: E402
from paper_2007_13552_b200 import _lib  # noqa: E402

comm = dnd.Communicator(0)
x = dnd.random_uniform((5_000_000, 18), 0, 42, comm)
for it in (1, 2, 5, 20):
    dnd.kmeans_fit(x, 8, it, 0.0, 42)
    torch.cuda.synchronize()
    t = (C.c_ulonglong * 16)()
    _lib.check(_lib.lib().dndc_internal_tail_trace(t))
    base = t[5]
    print(f"fit {it:2d} iters, last launch: cta0 start 0 | cta0 tail entry {(t[0]-base)/1e3:7.1f} us | last CTA "
          f"{(t[1]-base)/1e3:7.1f} | reduced {(t[2]-base)/1e3:7.1f} | exchanged {(t[3]-base)/1e3:7.1f} | "
          f"updated {(t[4]-base)/1e3:7.1f} [fold {(t[6]-t[3])/1e3:.1f} elem {(t[7]-t[6])/1e3:.1f} "
          f"clusters {(t[8]-t[7])/1e3:.1f} final {(t[4]-t[8])/1e3:.1f}]")

import numpy as np  # noqa: E402

ct = (C.c_ulonglong * 4096)()
_lib.check(_lib.lib().dndc_internal_cta_trace(ct))
a = np.array(ct[:], dtype=np.int64).reshape(2048, 2)
G = int((a[:, 0] > 0).sum())
a = a[:G]
st, en = (a[:, 0] - a[:, 0].min()) / 1e3, (a[:, 1] - a[:, 0].min()) / 1e3
print(f"{G} CTAs: start spread {st.max():.1f} us; finish min {en.min():.1f} p10 {np.percentile(en, 10):.1f} "
      f"median {np.median(en):.1f} p90 {np.percentile(en, 90):.1f} max {en.max():.1f} us")
sm = np.arange(G) % 148
late = np.argsort(en)[-8:]
print("latest CTAs (id, finish us):", [(int(i), round(float(en[i]), 1)) for i in late])

it = (C.c_ulonglong * 128)()
_lib.check(_lib.lib().dndc_internal_iter_trace(it))
v = np.array(it[:], dtype=np.int64).reshape(64, 2)[:20]
print("per iteration (us): kernel start->update done | gap to the next kernel's start")
print(" ".join(f"{(v[i,1]-v[i,0])/1e3:.0f}|{(v[i+1,0]-v[i,1])/1e3:.1f}" for i in range(19)))
