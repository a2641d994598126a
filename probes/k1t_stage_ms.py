"""Per-launch times (CUDA events, block_precond profile mode) of one config's apply, for K1t
experiments selected through environment switches. usage: k1t_stage_ms.py CONFIG [BATCH]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1712_00403_b200 as fdp, synth
cid = int(sys.argv[1])
w = synth.CONFIGS[cid]
batch = int(sys.argv[2]) if len(sys.argv) > 2 else w.batch
gd = fdp.discretization(w.dim, w.disc, w.p, w.n_el)
P = fdp.build_block(gd)
r = torch.randn(batch, gd.n_total, dtype=torch.float64, device="cuda"); s = torch.empty_like(r)
ws = P.workspace(batch)
for _ in range(2):
    P.apply(r, s, batch=batch, workspace=ws)
torch.cuda.synchronize()
P.profile(True)
for _ in range(3):
    P.apply(r, s, batch=batch, workspace=ws)
torch.cuda.synchronize()
prof = P.profile_read(); P.profile(False)
rows = prof
tot = sum(p[1] for p in rows)
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("FDP_"))
print(f"cfg {cid} [{tag}] total {tot:.3f} ms:", " ".join(f"{p[0]}:{p[1]:.3f}" for p in rows), flush=True)
