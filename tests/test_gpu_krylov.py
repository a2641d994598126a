"""NEXT-1: GPU-resident P_D-MINRES with libfdp's matrix-free Kronecker Stokes
operator. Parity against the oracle: the Kronecker operator (rectangular factors, accumulating
epilogue), the full Stokes operator (configs 1-3, ν = 1 and config 3's variable ν), the vector
kernels, and MINRES iteration counts (GPU operator + GPU P_D vs oracle operator + oracle P_D)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1712_00403_b200 as fdp  # noqa: E402
import synth  # noqa: E402
from paper_1712_00403_b200 import krylov  # noqa: E402
from oracle import kron as okron  # noqa: E402
from oracle import minres as ominres  # noqa: E402
from oracle import precond as oprec  # noqa: E402
from oracle import spaces as ospaces  # noqa: E402
from oracle import stokes as ostokes  # noqa: E402

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("nin,nout", [((5, 7, 3), (4, 9, 6)), ((65, 33, 9), (35, 40, 9)),
                                      ((120, 3, 5), (7, 130, 2)), ((6, 11), (13, 4))])
def test_kron_op_rectangular_terms(nin, nout):
    rng = np.random.default_rng(len(nin) + nin[0])
    terms = [[rng.standard_normal((o, i)) for i, o in zip(nin, nout)] for _ in range(3)]
    coef = [1.5, -0.25, 2.0]
    op = fdp.KronOp(terms, coef)
    x = rng.standard_normal((2, int(np.prod(nin))))
    y0 = rng.standard_normal((2, int(np.prod(nout))))
    X = dev(x)
    Y = dev(y0)
    op.apply(X, Y, alpha=0.5, beta=-2.0, batch=2, xbs=x.shape[1], ybs=y0.shape[1])
    for b in range(2):
        ref = -2.0 * y0[b] + 0.5 * sum(c * okron.kron_matvec(list(reversed(T)), x[b]) for c, T in zip(coef, terms))
        assert rel(Y[b].cpu().numpy(), ref) < 1e-13


@pytest.mark.parametrize("nin,nout,bw", [((130, 9, 7), (128, 9, 5), 5), ((9, 200, 6), (11, 190, 6), 9),
                                         ((7, 5, 300), (6, 4, 301), 3)])
def test_kron_op_banded_factors(nin, nout, bw):
    """Banded factors (K4 path: nonzeros in a band of width <= bw around a skewed diagonal, the
    B-spline Gram / mixed-matrix pattern) on the single and the grouped apply, vs the oracle."""
    rng = np.random.default_rng(sum(nin) + bw)

    def banded(o, i):
        F = rng.standard_normal((o, i))
        for a in range(o):
            c = int(round(a * (i - 1) / max(o - 1, 1)))
            lo, hi = max(0, c - bw // 2), min(i, c - bw // 2 + bw)
            F[a, :lo] = 0.0
            F[a, hi:] = 0.0
        return F

    terms = [[banded(o, i) for i, o in zip(nin, nout)] for _ in range(2)]
    coef = [0.75, -1.25]
    op = fdp.KronOp(terms, coef)
    x = rng.standard_normal(int(np.prod(nin)))
    y0 = rng.standard_normal(int(np.prod(nout)))
    ref = 0.5 * y0 + 2.0 * sum(c * okron.kron_matvec(list(reversed(T)), x) for c, T in zip(coef, terms))
    Y = dev(y0)
    op.apply(dev(x), Y, alpha=2.0, beta=0.5)
    assert rel(Y.cpu().numpy(), ref) < 1e-13
    Y = dev(y0)
    fdp.KronOp.apply_group([op], [dev(x)], [Y], [2.0], beta=0.5)
    assert rel(Y.cpu().numpy(), ref) < 1e-13


def test_kron_ops_grouped_matches_single():
    """kron_ops_apply: shared outputs accumulate, distinct outputs stay separate, beta applies once."""
    rng = np.random.default_rng(11)
    shapes = [((9, 70, 5), (9, 70, 5)), ((9, 70, 5), (8, 66, 5)), ((12, 7, 33), (9, 70, 5)),
              ((9, 70, 5), (3, 4, 5))]
    ops, xs, ys = [], [], []
    for nin, nout in shapes:
        nt = int(rng.integers(1, 4))
        terms = [[rng.standard_normal((o, i)) for i, o in zip(nin, nout)] for _ in range(nt)]
        ops.append((fdp.KronOp(terms, list(rng.standard_normal(nt))), terms))
        xs.append(rng.standard_normal(int(np.prod(nin))))
    y0 = rng.standard_normal(9 * 70 * 5), rng.standard_normal(8 * 66 * 5), rng.standard_normal(60)
    out_of = [0, 1, 0, 2]
    alphas = [0.5, -1.0, 2.0, 1.5]
    Y = [dev(v) for v in y0]
    fdp.KronOp.apply_group([o for o, _ in ops], [dev(x) for x in xs], [Y[k] for k in out_of], alphas,
                           beta=-0.75)
    for k in range(3):
        ref = -0.75 * y0[k]
        for i, (op, terms) in enumerate(ops):
            if out_of[i] == k:
                ref = ref + alphas[i] * sum(c * okron.kron_matvec(list(reversed(T)), xs[i])
                                            for c, T in zip(np.asarray(_coef(op)), terms))
        assert rel(Y[k].cpu().numpy(), ref) < 1e-13, k


def _coef(op):
    return op._coef


@pytest.mark.parametrize("band", [None, "1", "0"])
@pytest.mark.parametrize("cid", [1, 2, 3])
def test_stokes_operator_matches_oracle(cid, band, monkeypatch):
    """The GPU Stokes operator (grouped and per-operator) vs the oracle's; band: the banded K4
    factors forced on ("1", every factor of these configs is banded) or off ("0")."""
    if band is not None:
        monkeypatch.setenv("FDP_KRON_BAND", band)
    w = synth.CONFIGS[cid]
    nu_o = ostokes.config3_nu_terms(w.dim) if w.variable_nu else None
    nu_g = synth.viscosity_separable(w.dim) if w.variable_nu else None
    op = ostokes.StokesCube(w.dim, w.disc, w.p, w.n_el, nu_terms=nu_o)
    gop = krylov.StokesOperator(w.dim, w.disc, w.p, w.n_el, nu_terms=nu_g)
    assert gop.n == op.n
    x = np.random.default_rng(cid).standard_normal(op.n)
    y = torch.empty(op.n, dtype=torch.float64, device="cuda")
    ref = op.matvec(x)
    for grouped in (True, False):
        gop.grouped = grouped
        gop._apply_direct(dev(x), y)
        for k in range(len(op.sizes)):
            a, b = op.off_idx[k], op.off_idx[k + 1]
            assert rel(y[a:b].cpu().numpy(), ref[a:b]) < 1e-12, (grouped, k)


def test_vector_kernels():
    rng = np.random.default_rng(3)
    x, y, z = rng.standard_normal((3, 1_000_003))
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    fdp.vec_dot(dev(x), dev(y), out)
    assert abs(out.item() - x @ y) < 1e-12 * np.abs(x * y).sum()
    o = torch.empty(x.size, dtype=torch.float64, device="cuda")
    fdp.vec_lincomb(2.0, dev(x), -1.0, dev(y), 0.5, dev(z), o)
    assert np.max(np.abs(o.cpu().numpy() - (2 * x - y + 0.5 * z))) < 1e-14 * 10


@pytest.mark.parametrize("cid", [1, 2, 3])
def test_gpu_minres_iteration_counts(cid):
    """Whole P_D-MINRES on the GPU (libfdp operator, preconditioner and vector kernels) vs the
    oracle's MINRES with the oracle operator and P_D: identical iteration counts."""
    w = synth.CONFIGS[cid]
    nu_o = ostokes.config3_nu_terms(w.dim) if w.variable_nu else None
    nu_g = synth.viscosity_separable(w.dim) if w.variable_nu else None
    op = ostokes.StokesCube(w.dim, w.disc, w.p, w.n_el, nu_terms=nu_o)
    od = ospaces.build(w.dim, w.disc, w.p, w.n_el)
    gd = fdp.discretization(w.dim, w.disc, w.p, w.n_el)
    dv = dq = None
    if w.variable_nu:
        dv, dq = ospaces.nu_scalings(od, synth.viscosity)
    f = ostokes.project_rhs(synth.rhs(w.seed, op.n, 1)[0], op.sizes[-1])
    x_o, it_o, h_o = ominres.minres(op.matvec, f, oprec.BlockPrecond(od, dv, dq).apply)

    gop = krylov.StokesOperator(w.dim, w.disc, w.p, w.n_el, nu_terms=nu_g)
    P = fdp.build_block(gd, dscale_vel=dv, dscale_pres=dq)
    ws = P.workspace(1)
    x_g, it_g, h_g = krylov.minres(gop.apply, lambda r, z: P.apply(r, z, workspace=ws), dev(f))
    assert it_g == it_o, (cid, it_g, it_o)
    n = min(len(h_o), len(h_g))
    assert max(abs(a - b) / a for a, b in zip(h_o[:n], h_g[:n])) < 1e-6
    assert rel(x_g.cpu().numpy(), x_o) < 1e-6


@pytest.mark.parametrize("cid", [1, 2, 3])
def test_gpu_minres_device_resident(cid):
    """minres_device (scalar recurrence on the GPU, 6 iterations per graph replay): the oracle's
    iteration count, its residual history, and the host-driven GPU MINRES's solution."""
    w = synth.CONFIGS[cid]
    nu_o = ostokes.config3_nu_terms(w.dim) if w.variable_nu else None
    nu_g = synth.viscosity_separable(w.dim) if w.variable_nu else None
    op = ostokes.StokesCube(w.dim, w.disc, w.p, w.n_el, nu_terms=nu_o)
    od = ospaces.build(w.dim, w.disc, w.p, w.n_el)
    gd = fdp.discretization(w.dim, w.disc, w.p, w.n_el)
    dv = dq = None
    if w.variable_nu:
        dv, dq = ospaces.nu_scalings(od, synth.viscosity)
    f = ostokes.project_rhs(synth.rhs(w.seed, op.n, 1)[0], op.sizes[-1])
    x_o, it_o, h_o = ominres.minres(op.matvec, f, oprec.BlockPrecond(od, dv, dq).apply)
    gop = krylov.StokesOperator(w.dim, w.disc, w.p, w.n_el, nu_terms=nu_g)
    P = fdp.build_block(gd, dscale_vel=dv, dscale_pres=dq)
    ws = P.workspace(1)
    ap = lambda r, z: P.apply(r, z, workspace=ws)
    for _ in range(2):  # second call replays the captured graph
        x_g, it_g, h_g = krylov.minres_device(gop._apply_direct, ap, dev(f))
        assert it_g == it_o, (cid, it_g, it_o)
        assert max(abs(a - b) / a for a, b in zip(h_o, h_g)) < 1e-6
        assert rel(x_g.cpu().numpy(), x_o) < 1e-6
    x_h, it_h, _ = krylov.minres(gop.apply, ap, dev(f))
    assert it_h == it_g and rel(x_g.cpu().numpy(), x_h.cpu().numpy()) < 1e-10


def test_config3_paper_scalings_and_minres():
    """Config 3 with the paper's definition of the P^G scalings (C-6b): D_V, D_Q from
    libfdp vs the oracle, the resulting P_D^G apply, and identical MINRES counts."""
    w = synth.CONFIGS[3]
    q = w.p + 7
    nu_o = ostokes.config3_nu_terms(w.dim)
    op = ostokes.StokesCube(w.dim, w.disc, w.p, w.n_el, nu_terms=nu_o)
    od = ospaces.build(w.dim, w.disc, w.p, w.n_el)
    dv_o, dq_o = ostokes.nu_scalings_paper(od, op, synth.viscosity, q)
    gop = krylov.StokesOperator(w.dim, w.disc, w.p, w.n_el, nu_terms=synth.viscosity_separable(w.dim))
    gd = fdp.discretization(w.dim, w.disc, w.p, w.n_el)
    dv_g, dq_g = krylov.nu_scalings_paper(gd, gop, synth.viscosity, q)
    assert rel(dv_g, dv_o) < 1e-12 and rel(dq_g, dq_o) < 1e-12
    P = fdp.build_block(gd, dscale_vel=dv_g, dscale_pres=dq_g)
    oP = oprec.BlockPrecond(od, dv_o, dq_o)
    r = synth.rhs(w.seed, op.n, 1)[0]
    assert rel(P.apply(dev(r)).cpu().numpy(), oP.apply(r)) < 1e-9
    f = ostokes.project_rhs(r, op.sizes[-1])
    _, it_o, _ = ominres.minres(op.matvec, f, oP.apply)
    ws = P.workspace(1)
    _, it_g, _ = krylov.minres(gop.apply, lambda a, z: P.apply(a, z, workspace=ws), dev(f))
    assert it_g == it_o, (it_g, it_o)
    with open("gpurun_out/minres_counts.jsonl" if __import__("os").path.isdir("gpurun_out") else "/dev/null", "a") as fh:
        fh.write('{"config": 3, "scalings": "paper (diag ratios)", "iterations": %d}\n' % it_g)


def test_config3_literal_c3_minres():
    """Config 3 under the literal 'C^3' own-direction reading (C-3, secondary row):
    operator, P_D^G and MINRES all on the alpha_own = p - 1 spaces; identical counts."""
    w = synth.CONFIGS[3]
    a = w.p - 1
    op = ostokes.StokesCube(w.dim, w.disc, w.p, w.n_el, nu_terms=ostokes.config3_nu_terms(w.dim),
                            rt_own_alpha=a)
    od = ospaces.build(w.dim, w.disc, w.p, w.n_el, rt_own_alpha=a)
    gd = fdp.discretization(w.dim, w.disc, w.p, w.n_el, rt_own_alpha=a)
    assert op.vel_dims == [c.dims for c in od.comps] and gd.comp_dims == op.vel_dims
    dv, dq = ospaces.nu_scalings(od, synth.viscosity)
    f = ostokes.project_rhs(synth.rhs(w.seed, op.n, 1)[0], op.sizes[-1])
    _, it_o, h_o = ominres.minres(op.matvec, f, oprec.BlockPrecond(od, dv, dq).apply)
    gop = krylov.StokesOperator(w.dim, w.disc, w.p, w.n_el, nu_terms=synth.viscosity_separable(w.dim),
                                rt_own_alpha=a)
    P = fdp.build_block(gd, dscale_vel=dv, dscale_pres=dq)
    ws = P.workspace(1)
    _, it_g, h_g = krylov.minres(gop.apply, lambda r, z: P.apply(r, z, workspace=ws), dev(f))
    assert it_g == it_o, (it_g, it_o)
    assert max(abs(x - y) / x for x, y in zip(h_o, h_g)) < 1e-6
    with open("gpurun_out/minres_counts.jsonl" if __import__("os").path.isdir("gpurun_out") else "/dev/null", "a") as fh:
        fh.write('{"config": 3, "reading": "literal C^3 own direction", "iterations": %d}\n' % it_g)
