"""Small driver for ncu: cfg1 input, one 3-iteration fit (the assign kernel is
the capture target: -k regex:kmeans_assign)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2007_13552_b200.api as dnd

comm = dnd.Communicator(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 18
k = int(sys.argv[3]) if len(sys.argv) > 3 else 8
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 3
x = dnd.random_uniform((n, m), 0, 42, comm)
model = dnd.kmeans_fit(x, k, iters, 0.0, 42)
torch.cuda.synchronize()
print("inertia", model.inertia_trace)
