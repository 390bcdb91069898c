import sys, numpy as np
sys.path.insert(0, '.')
import paper_2007_13552_b200.api as dnd
from oracle.bind import Oracle
O = Oracle(); comm = dnd.Communicator(0)
for n, m in [(300, 130), (300, 96), (300, 97), (128, 130), (300, 64)]:
    xh = O.uniform_f32(n, m, 1000 + n)
    d = dnd.gather(dnd.cdist(dnd.from_global(xh, (n, m), 0, comm)))
    ref = O.cdist(xh.astype(np.float64))
    bad = np.argwhere(~np.isfinite(d))
    print(n, m, "nonfinite", len(bad), bad[:5].tolist(), "maxdev", np.nanmax(np.abs(d - ref)))
