"""Kernel-path experiments (not the bench): time block_precond_apply for a config under several
batch sizes and FDP_* environment switches; prints one line per variant. Diagnostic only."""
import os
import sys
import json

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1712_00403_b200 as fdp
import synth


def run(cid, batch, iters=50):
    w = synth.CONFIGS[cid]
    gd = fdp.discretization(w.dim, w.disc, w.p, w.n_el)
    dv = dq = None
    if w.variable_nu:
        dv, dq = fdp.nu_scalings(gd, synth.viscosity_separable(gd.D))
    P = fdp.build_block(gd, dscale_vel=dv, dscale_pres=dq)
    r = torch.randn(batch, gd.n_total, dtype=torch.float64, device="cuda")
    s = torch.empty_like(r)
    ws = P.workspace(batch)
    for _ in range(5):
        P.apply(r, s, batch=batch, workspace=ws)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        P.apply(r, s, batch=batch, workspace=ws)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / iters
    P.profile(True)
    P.apply(r, s, batch=batch, workspace=ws)
    torch.cuda.synchronize()
    P.apply(r, s, batch=batch, workspace=ws)
    torch.cuda.synchronize()
    prof = P.profile_read()
    P.profile(False)
    return ms, prof, P.launch_count(batch)


if __name__ == "__main__":
    cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    batches = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1", "4"])]
    variants = [{}, {"FDP_NO_FUSE": "1"}, {"FDP_NO_SMALL": "1"}]
    if len(sys.argv) > 3:
        variants = json.loads(sys.argv[3])
    for var in variants:
        for k in list(os.environ):
            if k.startswith("FDP_"):
                os.environ.pop(k, None)
        os.environ.update(var)
        for bt in batches:
            ms, prof, nl = run(cid, bt)
            per = [round(p[1] * 1e3, 1) for p in prof]
            fl = sum(p[2] for p in prof if p[0] == 0)
            k1ms = sum(p[1] for p in prof if p[0] == 0)
            print(json.dumps({"cfg": cid, "batch": bt, "env": var, "us_per_call": round(ms * 1e3, 1),
                              "us_per_rhs": round(ms * 1e3 / bt, 1), "launches": nl,
                              "profiled_us": per, "k1_tflops_profiled": round(fl / (k1ms * 1e-3) / 1e12, 2)}),
                  flush=True)
