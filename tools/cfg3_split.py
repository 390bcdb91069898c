"""cfg3 shard (6.25M x 64, k=64): fit iteration vs predict-only (no accumulation)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_13552_b200.api as dnd  # noqa: E402

comm = dnd.Communicator(0)
n, m, k = 6_250_000, 64, 64
x = dnd.random_uniform((n, m), 0, 42, comm)
model = dnd.kmeans_fit(x, k, 2, 0.0, 42)
print(f"refined rows in a 2-iteration fit: {model.refined_rows} ({model.refined_rows / (2 * n):.2%} of row-visits)")
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for label, fn in (("fit 20 it", lambda: dnd.kmeans_fit(x, k, 20, 0.0, 42)), ("predict", lambda: dnd.kmeans_predict(model, x))):
    fn()
    torch.cuda.synchronize()
    s.record()
    fn()
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e)
    per = t / 20 if label.startswith("fit") else t
    print(f"{label:10s} {t:8.2f} ms  per-iteration/pass {per:.3f} ms  {4.0*n*m/(per*1e-3)/1e9:.0f} GB/s", flush=True)
