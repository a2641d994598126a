"""End-to-end example: solve the Stokes system of BASELINE.json config 2 (unit cube, Taylor-Hood,
pressure degree 3, 32^3 elements) with P_D-MINRES, every vector operation on the GPU.

    python examples/solve_stokes.py [config]

The right-hand side is the config's seeded N(0,1) vector with its pressure part projected to zero
mean (the system is singular in the constant pressure). Prints iterations, solve time and the true
relative residual."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1712_00403_b200 as fdp
import synth
from paper_1712_00403_b200 import krylov

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = synth.CONFIGS[cid]
d = fdp.discretization(w.dim, w.disc, w.p, w.n_el)                  # pencils of P_V,k and P_Q
dv = dq = None
if w.variable_nu:                                                   # config 3: P_D^G scalings
    dv, dq = fdp.nu_scalings(d, synth.viscosity_separable(d.D))
P = fdp.build_block(d, dscale_vel=dv, dscale_pres=dq)               # libfdp handles
A = krylov.StokesOperator(w.dim, w.disc, w.p, w.n_el,
                          nu_terms=synth.viscosity_separable(w.dim) if w.variable_nu else None)
f = synth.rhs(w.seed, A.n, 1)[0]
f[-A.sizes[-1]:] -= f[-A.sizes[-1]:].mean()
b = torch.from_numpy(f).cuda()
ws = P.workspace(1)
precond = lambda r, z: P.apply(r, z, workspace=ws)

x, its, hist = krylov.minres_device(A._apply_direct, precond, b)    # warm-up (graph capture)
torch.cuda.synchronize()
t0 = time.perf_counter()
x, its, hist = krylov.minres_device(A._apply_direct, precond, b)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
r = torch.empty_like(x)
A.apply(x, r)
res = float(torch.linalg.norm(r - b) / torch.linalg.norm(b))
print(f"config {cid}: {A.n} dofs, {its} P_D-MINRES iterations, {dt * 1e3:.1f} ms, "
      f"true relative residual {res:.2e}")
