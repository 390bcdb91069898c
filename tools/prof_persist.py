"""One cfg1 fit for ncu (the persistent k-means kernel is one launch per fit).

    ncu --set full -k regex:persist -s 2 -c 1 python tools/prof_persist.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_13552_b200.api as dnd  # noqa: E402

comm = dnd.Communicator(0)
x = dnd.random_uniform((5_000_000, 18), 0, 42, comm)
for _ in range(4):
    m = dnd.kmeans_fit(x, 8, 20, 0.0, 42)
print("inertia", m.inertia_trace[-1])
