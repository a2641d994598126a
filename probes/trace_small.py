"""Per-warp phase timing of the small-n kernel launches of one block apply (diagnostic)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1712_00403_b200 as fdp
import synth

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1
w = synth.CONFIGS[cid]
gd = fdp.discretization(w.dim, w.disc, w.p, w.n_el)
P = fdp.build_block(gd)
r = torch.randn(batch, gd.n_total, dtype=torch.float64, device="cuda")
s = torch.empty_like(r)
ws = P.workspace(batch)
for _ in range(3):  # warm (graph captured without trace)
    P.apply(r, s, batch=batch, workspace=ws)
torch.cuda.synchronize()
cap = 1 << 22
buf = torch.zeros(cap, dtype=torch.int64, device="cuda")
fdp.lib.fdp_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
fdp.lib.fdp_debug_trace(buf.data_ptr(), cap)
s2 = torch.empty_like(r)  # new pointer -> re-capture with trace
P.apply(r, s2, batch=batch, workspace=ws)
torch.cuda.synchronize()
if "cold" in sys.argv:  # flush L2 (512 MB written + read back) before the traced apply
    fb = torch.empty(512 << 20 >> 2, dtype=torch.int32, device="cuda")
    fb.zero_()
    torch.sum(fb, dtype=torch.int64)
P.apply(r, s2, batch=batch, workspace=ws)  # replay (trace overwritten)
torch.cuda.synchronize()
fdp.lib.fdp_debug_trace(None, 0)
t = buf.cpu().numpy().astype(np.int64)
nl = P.launch_count(batch)
per = 148 * 16 * 6
t0g = None
for L in range(nl):
    a = t[L * per:(L + 1) * per].reshape(148 * 16, 6)
    valid = a[:, 0] > 0
    if not valid.any():
        continue
    a = a[valid]
    if t0g is None:
        t0g = a[:, 0].min()
    done = a[:, 5] > 0
    rel = (a - a[:, :1].min()) / 1e3
    print(f"launch {L}: start {(a[:,0].min()-t0g)/1e3:7.2f} us  span {(a[done,5].max()-a[:,0].min())/1e3:6.2f} us  warps {len(a)} with tile {done.sum()}")
    for ph, name in [(1, "W issue+pdl wait"), (2, "W wait+sync"), (3, "panel load"), (4, "compute"), (5, "epilogue")]:
        d = (a[done, ph] - a[done, ph - 1]) / 1e3
        print(f"    {name:18s} med {np.median(d):6.2f}  p10 {np.percentile(d,10):6.2f}  p90 {np.percentile(d,90):6.2f}  max {d.max():6.2f}")
    print(f"    first-tile end (rel) med {np.median(rel[done,5]):6.2f} max {rel[done,5].max():6.2f}; start spread {rel[:,0].max():6.2f}")
