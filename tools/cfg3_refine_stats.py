"""Near-tie rows per iteration of the cfg3 shard fit (6.25M x 64, k=64):
refined_rows of fits stopped after 1, 2, ... iterations (differences = the
iteration's queue length)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_13552_b200.api as dnd  # noqa: E402

comm = dnd.Communicator(0)
x = dnd.random_uniform((6_250_000, 64), 0, 42, comm)
prev = 0
for it in list(range(1, 9)) + [20]:
    m = dnd.kmeans_fit(x, 64, it, 0.0, 42)
    print(f"iterations {it:2d}: refined {m.refined_rows:8d}  (+{m.refined_rows - prev})", flush=True)
    prev = m.refined_rows
