import os, sys, hashlib
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2007_13552_b200.api as dnd
comm = dnd.Communicator(0)
x = dnd.random_uniform((2_000_000, 64), 0, 42, comm)
m = dnd.kmeans_fit(x, 64, 6, 0.0, 42)
print(os.environ.get("DNDC_LIB_PATH"), hashlib.sha1(np.ascontiguousarray(m.centroids).tobytes()).hexdigest(), repr(m.inertia_trace[-1]))
