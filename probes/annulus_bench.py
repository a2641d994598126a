"""GPU P_D- vs P_D^G-MINRES on the eighth of the thick annulus (NEXT-3, Table 3 setting:
TH, nu = 1; synthetic N(0,1) RHS with the pressure part projected)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_1712_00403_b200 import geometry as ggeo
from paper_1712_00403_b200 import krylov

cases = [(int(a), int(b)) for a, b in (c.split("x") for c in (sys.argv[1].split(",") if len(sys.argv) > 1 and "x" in sys.argv[1] else ["2x8", "3x16", "3x32"]))]
for p, n_el in cases:
    t0 = time.perf_counter()
    gop = ggeo.AnnulusStokesOperator(p, n_el)
    t_op = time.perf_counter() - t0
    f = np.random.default_rng(0).standard_normal(gop.n)
    f[-gop.sizes[-1]:] -= f[-gop.sizes[-1]:].mean()
    fd_ = torch.from_numpy(f).cuda()
    for name in ("P_D", "P_D^G"):
        t0 = time.perf_counter()
        P = ggeo.plain_block(gop) if name == "P_D" else ggeo.geometry_block(gop)[0]
        t_setup = time.perf_counter() - t0
        ws = P.workspace(1)
        ap = lambda r, z: P.apply(r, z, workspace=ws)
        krylov.minres(gop.apply, ap, fd_)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        x, its, _ = krylov.minres(gop.apply, ap, fd_)
        b.record()
        torch.cuda.synchronize()
        y = torch.empty_like(x)
        gop.apply(x, y)
        res = float(torch.linalg.norm(y - fd_) / torch.linalg.norm(fd_))
        print(json.dumps({"geometry": "eighth_annulus", "disc": "TH", "p": p, "n_el": n_el,
                          "dofs": gop.n, "precond": name, "iterations": its,
                          "gpu_solve_ms": a.elapsed_time(b), "true_rel_residual": res,
                          "setup_s": t_setup, "operator_setup_s": t_op}))


# P_T^G / P_C^G GMRES on the annulus (the paper's Tables 5-6 setting)
if "--gmres" in sys.argv:
    for p, n_el in cases:
        gop = ggeo.AnnulusStokesOperator(p, n_el)
        f = np.random.default_rng(0).standard_normal(gop.n)
        f[-gop.sizes[-1]:] -= f[-gop.sizes[-1]:].mean()
        fd_ = torch.from_numpy(f).cuda()
        P, _ = ggeo.geometry_block(gop)
        for variant in ("T", "C"):
            tri = P.tri(variant, gop.B, gop.BT)
            ws = tri.workspace()
            ap = lambda r, z: tri.apply(r, z, ws)
            krylov.gmres(gop.apply, ap, fd_)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            x, its, _ = krylov.gmres(gop.apply, ap, fd_)
            b.record()
            torch.cuda.synchronize()
            print(json.dumps({"geometry": "eighth_annulus", "disc": "TH", "p": p, "n_el": n_el,
                              "dofs": gop.n, "precond": f"P_{variant}^G", "solver": "GMRES",
                              "iterations": its, "gpu_solve_ms": a.elapsed_time(b)}))
