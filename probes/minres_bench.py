"""Time the GPU-resident P_D-MINRES (NEXT-1) per config against the oracle's CPU MINRES."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1712_00403_b200 as fdp
import synth
from paper_1712_00403_b200 import krylov

cids = [int(c) for c in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1", "2", "3"])]
oracle = "--oracle" in sys.argv
for cid in cids:
    w = synth.CONFIGS[cid]
    gd = fdp.discretization(w.dim, w.disc, w.p, w.n_el)
    dv = dq = None
    nu = synth.viscosity_separable(w.dim) if w.variable_nu else None
    if w.variable_nu:
        dv, dq = fdp.nu_scalings(gd, synth.viscosity_separable(gd.D))
    t0 = time.perf_counter()
    gop = krylov.StokesOperator(w.dim, w.disc, w.p, w.n_el, nu_terms=nu)
    P = fdp.build_block(gd, dscale_vel=dv, dscale_pres=dq)
    setup = time.perf_counter() - t0
    ws = P.workspace(1)
    f = synth.rhs(w.seed, gop.n, 1)[0]
    f[-gop.sizes[-1]:] -= f[-gop.sizes[-1]:].mean()
    fd_ = torch.from_numpy(f).cuda()
    x, its, _ = krylov.minres(gop.apply, lambda r, z: P.apply(r, z, workspace=ws), fd_)  # warm
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    x, its, _ = krylov.minres(gop.apply, lambda r, z: P.apply(r, z, workspace=ws), fd_)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    y = torch.empty_like(x)
    gop.apply(x, y)
    res = float(torch.linalg.norm(y - fd_) / torch.linalg.norm(fd_))
    # per-matvec and per-precond times
    a.record()
    for _ in range(10):
        gop.apply(x, y)
    b.record()
    torch.cuda.synchronize()
    mv = a.elapsed_time(b) / 10
    a.record()
    for _ in range(10):
        P.apply(x, y, workspace=ws)
    b.record()
    torch.cuda.synchronize()
    pc = a.elapsed_time(b) / 10
    # device-resident recurrence (6 iterations per graph replay); free the host-driven buffers
    krylov._BUFFERS.clear()
    torch.cuda.empty_cache()
    ap = lambda r, z: P.apply(r, z, workspace=ws)
    krylov.minres_device(gop._apply_direct, ap, fd_)
    torch.cuda.synchronize()
    a.record()
    xd, its_d, _ = krylov.minres_device(gop._apply_direct, ap, fd_)
    b.record()
    torch.cuda.synchronize()
    line = {"config": cid, "dofs": gop.n, "iterations": its, "gpu_solve_ms": ms, "true_rel_residual": res,
            "matvec_ms": mv, "precond_ms": pc, "setup_s": setup,
            "device_resident_iterations": its_d, "device_resident_solve_ms": a.elapsed_time(b)}
    if oracle:
        from oracle import minres as om, precond as op_, spaces as os_, stokes as ost
        odisc = os_.build(w.dim, w.disc, w.p, w.n_el)
        odv = odq = None
        if w.variable_nu:
            odv, odq = os_.nu_scalings(odisc, synth.viscosity)
        oop = ost.StokesCube(w.dim, w.disc, w.p, w.n_el, nu_terms=ost.config3_nu_terms(w.dim) if w.variable_nu else None)
        Po = op_.BlockPrecond(odisc, odv, odq)
        t0 = time.perf_counter()
        _, its_o, _ = om.minres(oop.matvec, f, Po.apply)
        line.update({"oracle_iterations": its_o, "oracle_solve_s": time.perf_counter() - t0,
                     "oracle_threads": os.cpu_count()})
    print(json.dumps(line), flush=True)
