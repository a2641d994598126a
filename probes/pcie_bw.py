"""Pinned host <-> device copy bandwidth at the config-2 vector size (e2e context)."""
import json
import torch
n = 866750
h = torch.randn(n, dtype=torch.float64).pin_memory()
o = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
for _ in range(3):
    d.copy_(h, non_blocking=True); o.copy_(d, non_blocking=True)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = {}
for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: o.copy_(d, non_blocking=True))]:
    a.record()
    for _ in range(20):
        fn()
    b.record()
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / 20
    res[name + "_us"] = t * 1e3
    res[name + "_GBs"] = n * 8 / (t * 1e-3) / 1e9
print(json.dumps(res))
