"""Config-2 apply time with a warm L2 vs after an L2 flush (write 512 MB, or write + read back),
per variant in one process (diagnostic for the bench's cold-L2 number)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_1712_00403_b200 as fdp
import synth

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = synth.CONFIGS[cid]
gd = fdp.discretization(w.dim, w.disc, w.p, w.n_el)
P = fdp.build_block(gd)
r = torch.randn(1, gd.n_total, dtype=torch.float64, device="cuda")
s = torch.empty_like(r)
ws = P.workspace(1)
buf = torch.empty(512 << 20 >> 2, dtype=torch.int32, device="cuda")
small = torch.empty(1 << 20, dtype=torch.int32, device="cuda")


def flush(kind):
    if kind == "write":
        buf.zero_()
    elif kind == "write+read":
        buf.zero_()
        torch.sum(buf, dtype=torch.int64)
    elif kind == "read":
        torch.sum(buf, dtype=torch.int64)
    elif kind == "small-kernel":
        small.zero_()


for kind in ["none", "small-kernel", "write", "write+read", "read", "none"]:
    for _ in range(5):
        flush(kind)
        P.apply(r, s, workspace=ws)
    torch.cuda.synchronize()
    ts = []
    for _ in range(50):
        flush(kind)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        P.apply(r, s, workspace=ws)
        b.record()
        ts.append((a, b))
    torch.cuda.synchronize()
    v = sorted(x.elapsed_time(y) * 1e3 for x, y in ts)
    print(f"{kind:14s} p10 {v[5]:6.1f}  p50 {v[25]:6.1f}  p90 {v[45]:6.1f} us", flush=True)
