"""Per-CTA phase timing of the plane kernel (and per-warp phases of the mode-1 passes) of one block
apply on the plane path (diagnostic)."""
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
cold = "cold" in sys.argv  # flush L2 (512 MB written + read back) before the traced apply
w = synth.CONFIGS[cid]
gd = fdp.discretization(w.dim, w.disc, w.p, w.n_el)
P = fdp.build_block(gd)
r = torch.randn(1, gd.n_total, dtype=torch.float64, device="cuda")
s = torch.empty_like(r)
ws = P.workspace(1)
for _ in range(3):
    P.apply(r, s, batch=1, workspace=ws)
torch.cuda.synchronize()
cap = 1 << 22
buf = torch.zeros(cap, dtype=torch.int64, device="cuda")
fdp.lib.fdp_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
fdp.lib.fdp_debug_trace(buf.data_ptr(), cap)
s2 = torch.empty_like(r)
P.apply(r, s2, batch=1, workspace=ws)
torch.cuda.synchronize()
if cold:
    fb = torch.empty(512 << 20 >> 2, dtype=torch.int32, device="cuda")
    fb.zero_()
    torch.sum(fb, dtype=torch.int64)
P.apply(r, s2, batch=1, workspace=ws)
torch.cuda.synchronize()
fdp.lib.fdp_debug_trace(None, 0)
t = buf.cpu().numpy().astype(np.int64)
nsm = torch.cuda.get_device_properties(0).multi_processor_count
small = nsm * 16 * 6
a0 = t[:small].reshape(-1, 6)
a0 = a0[a0[:, 0] > 0]
t0 = a0[:, 0].min()
print(f"L1 start 0, first-tile end max {(a0[a0[:,5]>0,5].max()-t0)/1e3:.2f} us")
grid = 2 * nsm
# plane launch: grid * 8 entries; find grid by scanning for the next small chunk
p = t[small:small + 8 * 2 * nsm].reshape(-1, 8)
valid = p[:, 0] > 0
p = p[valid]
names = ["start", "W+pdl", "plane load", "mode-2 fwd", "mode-3 fused", "mode-2 bwd", "store"]
print(f"L2 CTAs {len(p)}: start {(p[:,0].min()-t0)/1e3:.2f} .. {(p[:,0].max()-t0)/1e3:.2f} us, end max {(p[:,6].max()-t0)/1e3:.2f} us")
kind = p[:, 7] >> 32
smid = (p[:, 7] >> 16) & 0xFFFF
import collections
cnt = collections.Counter(smid.tolist())
per = collections.Counter(cnt.values())
print("  CTAs per SM:", dict(sorted(per.items())), " SMs used:", len(cnt))
two = [sm for sm, c in cnt.items() if c == 2]
one = [sm for sm, c in cnt.items() if c == 1]
for label, sms in (("SMs with 2 CTAs", two), ("SMs with 1 CTA", one)):
    sel = np.isin(smid, sms) & (kind == 0)
    if sel.any():
        print(f"  {label}: kind-0 end med {np.median((p[sel,6]-t0)/1e3):.2f} max {((p[sel,6]-t0)/1e3).max():.2f} us,"
              f" start med {np.median((p[sel,0]-t0)/1e3):.2f}")
for kd in (0, 1):
    q = p[kind == kd]
    if not len(q):
        continue
    print(f"  kind {kd}: {len(q)} CTAs")
    prev = 1
    for ph in range(2, 7):
        if kd == 1 and ph == 5:
            continue
        d = (q[:, ph] - q[:, prev]) / 1e3
        print(f"    {names[ph]:14s} med {np.median(d):6.2f} p10 {np.percentile(d,10):6.2f} p90 {np.percentile(d,90):6.2f} max {d.max():6.2f}")
        prev = ph
    print(f"    end (rel t0) med {np.median((q[:,6]-t0)/1e3):6.2f} max {((q[:,6]-t0)/1e3).max():6.2f}")
n2 = 8 * len(t[small:small + 8 * 2 * nsm].reshape(-1, 8))
a2 = t[small + 8 * len(valid):small + 8 * len(valid) + small].reshape(-1, 6)
a2 = a2[a2[:, 0] > 0]
if len(a2):
    print(f"L3 start {(a2[:,0].min()-t0)/1e3:.2f} us, first-tile end max {(a2[a2[:,5]>0,5].max()-t0)/1e3:.2f} us")
