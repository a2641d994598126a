"""NEXT-3: TH Stokes on the eighth of the thick annulus
with the geometry-aware P_D^G (§6, Appendix), through libfdp, against
oracle/geometry.py: the mapped operator, the P_D^G apply and identical MINRES iteration counts for
the plain and the geometry-aware preconditioner."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1712_00403_b200 import geometry as ggeo  # noqa: E402
from paper_1712_00403_b200 import krylov  # noqa: E402
from oracle import geometry as ogeo  # noqa: E402
from oracle import minres as ominres  # noqa: E402
from oracle import precond as oprec  # noqa: E402
from oracle import stokes as ostokes  # noqa: E402

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("p,n_el", [(1, 3), (2, 4), (3, 8)])
def test_annulus_operator_matches_oracle(p, n_el):
    op = ogeo.StokesMapped(ogeo.annulus(), p, n_el)
    gop = ggeo.AnnulusStokesOperator(p, n_el)
    assert gop.n == op.n and gop.sizes == [int(s) for s in op.sizes]
    x = np.random.default_rng(p).standard_normal(op.n)
    y = torch.empty(op.n, dtype=torch.float64, device="cuda")
    ref = op.matvec(x)
    for grouped in (True, False):
        gop.grouped = grouped
        gop._apply_direct(dev(x), y)
        for k in range(4):
            a, b = op.off_idx[k], op.off_idx[k + 1]
            assert rel(y[a:b].cpu().numpy(), ref[a:b]) < 1e-12, (grouped, k)


@pytest.mark.parametrize("p,n_el", [(2, 4), (3, 8)])
def test_geometry_aware_block_matches_oracle(p, n_el):
    op = ogeo.StokesMapped(ogeo.annulus(), p, n_el)
    disc, dv, dq = ogeo.geo_discretization(op)
    oP = oprec.BlockPrecond(disc, dv, dq)
    gop = ggeo.AnnulusStokesOperator(p, n_el)
    P, _ = ggeo.geometry_block(gop)
    r = np.random.default_rng(3).standard_normal(op.n)
    s = P.apply(dev(r)).cpu().numpy()
    ref = oP.apply(r)
    for k in range(4):
        a, b = op.off_idx[k], op.off_idx[k + 1]
        assert rel(s[a:b], ref[a:b]) < 1e-9, (k, rel(s[a:b], ref[a:b]))


@pytest.mark.parametrize("p,n_el", [(2, 8), (3, 8)])
def test_annulus_minres_iteration_counts(p, n_el):
    """GPU MINRES (libfdp operator + preconditioner) vs the oracle: identical counts for P_D and
    the geometry-aware P_D^G, and P_D^G needs far fewer."""
    op = ogeo.StokesMapped(ogeo.annulus(), p, n_el)
    f = ostokes.project_rhs(np.random.default_rng(0).standard_normal(op.n), op.sizes[-1])
    disc, dv, dq = ogeo.geo_discretization(op)
    _, it_po, _ = ominres.minres(op.matvec, f, oprec.BlockPrecond(ogeo.plain_discretization(op)).apply)
    _, it_go, _ = ominres.minres(op.matvec, f, oprec.BlockPrecond(disc, dv, dq).apply)
    gop = ggeo.AnnulusStokesOperator(p, n_el)
    counts = []
    for P in (ggeo.plain_block(gop), ggeo.geometry_block(gop)[0]):
        ws = P.workspace(1)
        _, it, _ = krylov.minres(gop.apply, lambda r, z: P.apply(r, z, workspace=ws), dev(f))
        counts.append(it)
    assert counts == [it_po, it_go], (counts, it_po, it_go)
    assert it_go < 0.8 * it_po


@pytest.mark.parametrize("variant", ["T", "C"])
def test_annulus_block_gmres_counts(variant):
    """P_T^G- / P_C^G-GMRES on the annulus (the paper's Tables 5-6 setting): identical counts."""
    from oracle import gmres as ogmres
    p, n_el = 2, 8
    op = ogeo.StokesMapped(ogeo.annulus(), p, n_el)
    f = ostokes.project_rhs(np.random.default_rng(0).standard_normal(op.n), op.sizes[-1])
    disc, dv, dq = ogeo.geo_discretization(op)
    oblk = oprec.BlockPrecond(disc, dv, dq)
    oP = (oprec.TriangularPrecond if variant == "T" else oprec.ConstrainedPrecond)(oblk, op)
    _, it_o, _ = ogmres.gmres(op.matvec, f, oP.apply)
    gop = ggeo.AnnulusStokesOperator(p, n_el)
    P, _ = ggeo.geometry_block(gop)
    tri = P.tri(variant, gop.B, gop.BT)
    ws = tri.workspace()
    _, it_g, _ = krylov.gmres(gop.apply, lambda r, z: tri.apply(r, z, ws), dev(f))
    assert it_g == it_o, (variant, it_g, it_o)
