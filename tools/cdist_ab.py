"""cfg2 cdist_xy with the FFMA panel kernel vs the tcgen05 path (env
DNDC_CDIST_TC_MIN_M), each in its own process, plus parity vs the oracle."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, torch, numpy as np
sys.path.insert(0, ".")
import paper_2007_13552_b200.api as dnd
from paper_2007_13552_b200 import _lib
from oracle.bind import Oracle
comm = dnd.Communicator(0)
n, m = 200_000, 18
x = dnd.random_uniform((n, m), 0, 42, comm); y = dnd.random_uniform((n, m), 0, 43, comm)
out = torch.empty((n, n), dtype=torch.float32, device="cuda")
L = _lib.lib()
run = lambda: _lib.check(L.dndc_cdist_xy_f32(comm.handle, x.tile.data_ptr(), n, y.tile.data_ptr(), n, m, out.data_ptr()))
run(); torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(3): run()
e.record(); torch.cuda.synchronize()
t = s.elapsed_time(e) / 3 / 1e3
O = Oracle()
rows = np.array([0, 1, 12345, 99999, 199999])
xh = O.uniform_f32(n, m, 42)[rows].astype(np.float64); yh = O.uniform_f32(n, m, 43).astype(np.float64)
ref = O.cdist_xy(xh, yh)
got = out[torch.from_numpy(rows).cuda()].cpu().numpy().astype(np.float64)
dev = float(np.max(np.abs(got - ref) / np.maximum(1, np.abs(ref))))
print(f"{t*1e3:.1f} ms  {4.0*n*n/t/1e9:.0f} GB/s  rel dev {dev:.2e}")
'''
import glob
runs = [("default", {}), ("ffma panel", {"DNDC_CDIST_TC_MIN_M": "100000"}), ("tcgen05 3xTF32", {"DNDC_CDIST_TC_MIN_M": "1"})]
runs += [(os.path.basename(v), {"DNDC_LIB_PATH": v}) for v in sorted(glob.glob(os.path.join(ROOT, "variants", "*.so")))]
for label, env in runs:
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=dict(os.environ, **env), capture_output=True,
                       text=True, timeout=600)
    print(f"{label:16s}", r.stdout.strip() or r.stderr.strip()[-500:], flush=True)
