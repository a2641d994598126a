"""NEXT-2: block-triangular P_T and constrained P_C through
libfdp's block_tri_apply, and GPU GMRES, against the oracle (oracle/precond.py, oracle/gmres.py):
element-wise parity of the preconditioner applies on configs 1-3 (config 3 with its P^G diagonal
scaling), the Arnoldi helper kernels, and identical GMRES iteration counts."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1712_00403_b200 as fdp  # noqa: E402
import synth  # noqa: E402
from paper_1712_00403_b200 import krylov  # noqa: E402
from oracle import gmres as ogmres  # noqa: E402
from oracle import precond as oprec  # noqa: E402
from oracle import spaces as ospaces  # noqa: E402
from oracle import stokes as ostokes  # noqa: E402

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _setup(cid):
    w = synth.CONFIGS[cid]
    nu_o = ostokes.config3_nu_terms(w.dim) if w.variable_nu else None
    nu_g = synth.viscosity_separable(w.dim) if w.variable_nu else None
    op = ostokes.StokesCube(w.dim, w.disc, w.p, w.n_el, nu_terms=nu_o)
    od = ospaces.build(w.dim, w.disc, w.p, w.n_el)
    gd = fdp.discretization(w.dim, w.disc, w.p, w.n_el)
    dv = dq = None
    if w.variable_nu:
        dv, dq = ospaces.nu_scalings(od, synth.viscosity)
    gop = krylov.StokesOperator(w.dim, w.disc, w.p, w.n_el, nu_terms=nu_g)
    P = fdp.build_block(gd, dscale_vel=dv, dscale_pres=dq)
    return w, op, oprec.BlockPrecond(od, dv, dq), gop, P


@pytest.mark.parametrize("cid", [1, 2, 3])
@pytest.mark.parametrize("variant", ["T", "C"])
def test_block_tri_matches_oracle(cid, variant):
    w, op, oblk, gop, P = _setup(cid)
    oP = (oprec.TriangularPrecond if variant == "T" else oprec.ConstrainedPrecond)(oblk, op)
    tri = P.tri(variant, gop.B, gop.BT)
    r = synth.rhs(w.seed, op.n, 1)[0]
    s = torch.empty(op.n, dtype=torch.float64, device="cuda")
    tri.apply(dev(r), s, tri.workspace())
    ref = oP.apply(r)
    got = s.cpu().numpy()
    for k in range(len(op.sizes)):
        a, b = op.off_idx[k], op.off_idx[k + 1]
        assert rel(got[a:b], ref[a:b]) < 1e-9, (k, rel(got[a:b], ref[a:b]))


def test_block_tri_rejects_mismatched_blocks():
    _, _, _, gop, P = _setup(1)
    with pytest.raises(fdp.FdpError):
        P.tri("T", gop.BT, gop.B)  # swapped: extents do not match


@pytest.mark.parametrize("m,n", [(1, 1000), (7, 12345), (37, 300001)])
def test_arnoldi_helpers(m, n):
    rng = np.random.default_rng(m)
    V = rng.standard_normal((m + 2, n))
    x = rng.standard_normal(n)
    Vd, xd = dev(V), dev(x)
    h = torch.zeros(m + 2, dtype=torch.float64, device="cuda")
    fdp.vec_multidot(Vd, m, xd, h)
    ref = V[:m] @ x
    assert np.max(np.abs(h[:m].cpu().numpy() - ref)) < 1e-12 * np.abs(V[:m]).sum(axis=1).max()
    assert np.all(h[m:].cpu().numpy() == 0.0)
    c = rng.standard_normal(m)
    hc = dev(c)
    y = xd.clone()
    fdp.vec_gemv(Vd, m, hc, -0.5, y, 2.0)
    assert np.max(np.abs(y.cpu().numpy() - (2.0 * x - 0.5 * V[:m].T @ c))) < 1e-12 * (np.abs(c).sum() + 2)


@pytest.mark.parametrize("cid", [1, 2, 3])
@pytest.mark.parametrize("variant", ["T", "C"])
def test_gpu_gmres_iteration_counts(cid, variant):
    """Whole P_T- / P_C-GMRES on the GPU vs the oracle's GMRES with the oracle operator and
    preconditioner: identical iteration counts, residual histories within rounding."""
    w, op, oblk, gop, P = _setup(cid)
    oP = (oprec.TriangularPrecond if variant == "T" else oprec.ConstrainedPrecond)(oblk, op)
    f = ostokes.project_rhs(synth.rhs(w.seed, op.n, 1)[0], op.sizes[-1])
    x_o, it_o, h_o = ogmres.gmres(op.matvec, f, oP.apply)
    tri = P.tri(variant, gop.B, gop.BT)
    ws = tri.workspace()
    x_g, it_g, h_g = krylov.gmres(gop.apply, lambda r, z: tri.apply(r, z, ws), dev(f))
    assert it_g == it_o, (cid, variant, it_g, it_o)
    assert max(abs(a - b) / a for a, b in zip(h_o, h_g)) < 1e-6
    nq = op.sizes[-1]
    xg = x_g.cpu().numpy()
    xg[-nq:] -= xg[-nq:].mean()
    x_o[-nq:] -= x_o[-nq:].mean()
    assert rel(xg, x_o) < 1e-6


@pytest.mark.parametrize("cid", [1, 2, 3])
@pytest.mark.parametrize("variant", ["T", "C"])
def test_gpu_gmres_device_resident(cid, variant):
    """gmres_device (Arnoldi bookkeeping on the GPU, 4 steps per graph replay): the oracle's
    iteration count and history, and the host-driven GPU GMRES's solution."""
    w, op, oblk, gop, P = _setup(cid)
    oP = (oprec.TriangularPrecond if variant == "T" else oprec.ConstrainedPrecond)(oblk, op)
    f = ostokes.project_rhs(synth.rhs(w.seed, op.n, 1)[0], op.sizes[-1])
    _, it_o, h_o = ogmres.gmres(op.matvec, f, oP.apply)
    tri = P.tri(variant, gop.B, gop.BT)
    ws = tri.workspace()
    ap = lambda r, z: tri.apply(r, z, ws)
    for _ in range(2):
        x_d, it_d, h_d = krylov.gmres_device(gop._apply_direct, ap, dev(f))
        assert it_d == it_o, (cid, variant, it_d, it_o)
        assert max(abs(a - b) / a for a, b in zip(h_o, h_d)) < 1e-6
    x_h, it_h, _ = krylov.gmres(gop.apply, ap, dev(f))
    assert it_h == it_d
    assert rel(x_d.cpu().numpy(), x_h.cpu().numpy()) < 1e-9
