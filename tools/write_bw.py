"""Pure-write, pure-read and copy bandwidth of this B200 (torch kernels, CUDA events):
the ceiling for cdist, whose traffic is almost all output writes."""
import json

import torch

n = 4 << 30  # floats (16 GB)
a = torch.empty(n, dtype=torch.float32, device="cuda")
b = torch.empty(n // 4, dtype=torch.float32, device="cuda")
c = torch.empty(n // 4, dtype=torch.float32, device="cuda")
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = {}
r = torch.empty(1, dtype=torch.float32, device="cuda")
for name, fn, byt in (("write_fill", lambda: a.fill_(1.0), 4.0 * n),
                      ("copy_rw", lambda: c.copy_(b), 2 * 4.0 * n / 4),
                      ("read_sum", lambda: torch.sum(a), 4.0 * n)):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    res[name + "_GBs"] = byt / best / 1e9
print(json.dumps(res))
