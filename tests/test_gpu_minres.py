"""MINRES iteration-count parity (BASELINE.json north_star: "preconditioned MINRES iteration
counts must be identical"): the oracle's MINRES on the oracle's Kronecker Stokes operator, run
once with the oracle's P_D (or P_D^G) and once with libfdp's block_precond_apply on the GPU.
RHS = the config's seeded N(0,1) vector with its pressure part projected off the null space
(SURVEY.md C-15); tolerance 1e-8, zero initial guess."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1712_00403_b200 as fdp  # noqa: E402
import synth  # noqa: E402
from oracle import minres, precond, spaces, stokes  # noqa: E402

pytestmark = pytest.mark.gpu


def _run(cid):
    w = synth.CONFIGS[cid]
    nu_terms = stokes.config3_nu_terms(w.dim) if w.variable_nu else None
    op = stokes.StokesCube(w.dim, w.disc, w.p, w.n_el, nu_terms=nu_terms)
    od = spaces.build(w.dim, w.disc, w.p, w.n_el)
    gd = fdp.discretization(w.dim, w.disc, w.p, w.n_el)
    dv = dq = None
    if w.variable_nu:
        dv, dq = spaces.nu_scalings(od, synth.viscosity)
    P_or = precond.BlockPrecond(od, dv, dq)
    P_gpu = fdp.build_block(gd, dscale_vel=dv, dscale_pres=dq)
    r_dev = torch.empty(gd.n_total, dtype=torch.float64, device="cuda")
    s_dev = torch.empty_like(r_dev)
    ws = P_gpu.workspace(1)

    def gpu_apply(r):
        r_dev.copy_(torch.from_numpy(r))
        P_gpu.apply(r_dev, s_dev, workspace=ws)
        return s_dev.cpu().numpy()

    f = stokes.project_rhs(synth.rhs(w.seed, op.n, 1)[0], op.sizes[-1])
    x1, it1, h1 = minres.minres(op.matvec, f, P_or.apply)
    x2, it2, h2 = minres.minres(op.matvec, f, gpu_apply)
    return it1, it2, h1, h2, x1, x2, op, f


@pytest.mark.parametrize("cid", [1, 2, 3])
def test_minres_iteration_counts_identical(cid):
    it1, it2, h1, h2, x1, x2, op, f = _run(cid)
    assert it1 == it2, (cid, it1, it2)
    assert it1 < 1000
    n = min(len(h1), len(h2))
    rel = max(abs(a - b) / a for a, b in zip(h1[:n], h2[:n]))
    assert rel < 1e-6, rel
    assert np.linalg.norm(x1 - x2) / np.linalg.norm(x1) < 1e-6
    res = np.linalg.norm(op.matvec(x2) - f) / np.linalg.norm(f)
    assert res < 1e-5
    import json, os
    if os.path.isdir("gpurun_out"):
        with open("gpurun_out/minres_counts.jsonl", "a") as fh:
            fh.write(json.dumps({"config": cid, "its_oracle_P": it1, "its_gpu_P": it2,
                                 "max_rel_hist_diff": rel, "true_rel_residual": res}) + "\n")
