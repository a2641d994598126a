"""Time GPU P_T-/P_C-GMRES (NEXT-2) per config: solve time, iterations, per-apply times."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_1712_00403_b200 as fdp
import synth
from paper_1712_00403_b200 import krylov

cids = [int(c) for c in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1", "2", "3"])]
for cid in cids:
    w = synth.CONFIGS[cid]
    gd = fdp.discretization(w.dim, w.disc, w.p, w.n_el)
    dv = dq = None
    nu = synth.viscosity_separable(w.dim) if w.variable_nu else None
    if w.variable_nu:
        dv, dq = fdp.nu_scalings(gd, synth.viscosity_separable(gd.D))
    gop = krylov.StokesOperator(w.dim, w.disc, w.p, w.n_el, nu_terms=nu)
    P = fdp.build_block(gd, dscale_vel=dv, dscale_pres=dq)
    f = synth.rhs(w.seed, gop.n, 1)[0]
    f[-gop.sizes[-1]:] -= f[-gop.sizes[-1]:].mean()
    fd_ = torch.from_numpy(f).cuda()
    for variant in ("T", "C"):
        tri = P.tri(variant, gop.B, gop.BT)
        ws = tri.workspace()
        r_buf = torch.empty(gop.n, dtype=torch.float64, device="cuda")
        z_buf = torch.empty_like(r_buf)
        graphs = {}

        def papply(r, z):
            key = (r.data_ptr(), z.data_ptr())
            g = graphs.get(key)
            if g is None:
                tri.apply(r, z, ws)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    tri.apply(r, z, ws)
                graphs[key] = g
            g.replay()
            return z

        x, its, _ = krylov.gmres(gop.apply, papply, fd_)  # warm
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        x, its, _ = krylov.gmres(gop.apply, papply, fd_)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        y = torch.empty_like(x)
        gop.apply(x, y)
        nq = gop.sizes[-1]
        res = float(torch.linalg.norm(y - fd_) / torch.linalg.norm(fd_))
        r_buf.copy_(fd_)
        papply(r_buf, z_buf)
        a.record()
        for _ in range(20):
            papply(r_buf, z_buf)
        b.record()
        torch.cuda.synchronize()
        pms = a.elapsed_time(b) / 20
        # device-resident Arnoldi bookkeeping (4 steps per graph replay)
        apd = lambda r, z: tri.apply(r, z, ws)
        krylov.gmres_device(gop._apply_direct, apd, fd_)
        torch.cuda.synchronize()
        a.record()
        xd, its_d, _ = krylov.gmres_device(gop._apply_direct, apd, fd_)
        b.record()
        torch.cuda.synchronize()
        print(json.dumps({"config": cid, "variant": variant, "dofs": gop.n, "iterations": its,
                          "gpu_solve_ms": ms, "true_rel_residual": res, "precond_ms": pms,
                          "device_resident_iterations": its_d,
                          "device_resident_solve_ms": a.elapsed_time(b)}))
