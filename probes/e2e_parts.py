"""Where does the host-buffer (e2e) time of config 2 go? Times the pieces on the device."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1712_00403_b200 as fdp
import synth

w = synth.CONFIGS[2]
gd = fdp.discretization(w.dim, w.disc, w.p, w.n_el)
P = fdp.build_block(gd)
f0 = P.fds[0]
x = torch.randn(f0.N, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
ws = torch.empty(f0.workspace_bytes(1) // 8 + 1, dtype=torch.float64, device="cuda")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def tm(fn, n=20):
    fn()
    torch.cuda.synchronize()
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


res = {"fd_one_component_us": tm(lambda: f0.apply(x, y, workspace=ws))}
r = torch.randn(gd.n_total, dtype=torch.float64, device="cuda")
s = torch.empty_like(r)
wsb = P.workspace(1)
res["block_apply_us"] = tm(lambda: P.apply(r, s, workspace=wsb))
rh = fdp.host_empty((1, gd.n_total))
rh[...] = r.cpu().numpy()
sh = fdp.host_empty((1, gd.n_total))
import time
P.apply_host(rh, sh)
t0 = time.perf_counter()
for _ in range(50):
    P.apply_host(rh, sh)
res["apply_host_us_wall"] = (time.perf_counter() - t0) / 50 * 1e6
print(json.dumps(res))
