"""BASELINE config 3's per-GPU shard (6.25M x 64 = 1/8 of 50M, k=64) for ncu:
two 20-iteration fits; profile a delta-iteration launch of kmeans_tc_kernel,
e.g.  ncu --set full -k kmeans_tc_kernel -s 25 -c 1 python tools/prof_cfg3.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_13552_b200.api as dnd  # noqa: E402

comm = dnd.Communicator(0)
x = dnd.random_uniform((6_250_000, 64), 0, 42, comm)
for _ in range(2):
    m = dnd.kmeans_fit(x, 64, 20, 0.0, 42)
print("inertia", m.inertia_trace[-1], "refined", m.refined_rows)
