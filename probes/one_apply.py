"""Run a few block_precond_apply calls of one config/batch (for ncu captures). Diagnostic only."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1712_00403_b200 as fdp
import synth

cid = int(sys.argv[1]); batch = int(sys.argv[2]); reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
w = synth.CONFIGS[cid]
gd = fdp.discretization(w.dim, w.disc, w.p, w.n_el)
P = fdp.build_block(gd)
r = torch.randn(batch, gd.n_total, dtype=torch.float64, device="cuda")
s = torch.empty_like(r)
ws = P.workspace(batch)
for _ in range(reps):
    P.apply(r, s, batch=batch, workspace=ws)
torch.cuda.synchronize()
print("ok", cid, batch)
