"""Time a 20-iteration k-means fit on BASELINE config 3's per-GPU shard
(6.25M x 64, k=64) and on the 5M slice: ms per iteration (CUDA events)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_13552_b200.api as dnd  # noqa: E402

comm = dnd.Communicator(0)
x = dnd.random_uniform((6_250_000, 64), 0, 42, comm)
dnd.kmeans_fit(x, 64, 20, 0.0, 42)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(3):
    m = dnd.kmeans_fit(x, 64, 20, 0.0, 42)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 3
print(f"cfg3 shard 6.25M x 64, k=64: {ms:.2f} ms per fit, {ms / 20:.3f} ms per iteration, "
      f"{6.25e6 * 64 * 4 * 20 / (ms * 1e-3) / 1e9:.0f} GB/s; inertia {m.inertia_trace[-1]!r}")
