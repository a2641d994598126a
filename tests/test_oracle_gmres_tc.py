"""Pins for the NEXT-2 oracle: GMRES (oracle/gmres.py, Saad & Schultz, PAPER.md
P:619) against the dense solve, the brute-force Krylov least-squares minimum and MINRES on
symmetric systems; the block-triangular P_T and constrained P_C against dense solves
with the explicitly assembled block matrices (not the factorization they are applied by)."""
import numpy as np
import pytest

from oracle import fd, gmres, minres, precond, spaces, stokes


def _nonsym(n, seed):
    rng = np.random.default_rng(seed)
    return np.eye(n) * 4 + rng.standard_normal((n, n)) / np.sqrt(n), rng.standard_normal(n)


def test_gmres_finite_termination_dense_solve():
    A, b = _nonsym(30, 1)
    x, it, hist = gmres.gmres(lambda v: A @ v, b, lambda v: v, tol=1e-14)
    assert it <= 30
    assert np.linalg.norm(x - np.linalg.solve(A, b)) < 1e-11 * np.linalg.norm(x)
    assert all(a >= b_ - 1e-15 for a, b_ in zip(hist, hist[1:]))  # residual never increases


def test_gmres_history_is_krylov_minimum():
    """||z_k|| = min over K_k(C, z_0) of ||z_0 - C y||, C = P^{-1} A, by brute-force least squares
    on the explicit (column-normalized) Krylov matrix."""
    A, b = _nonsym(40, 2)
    Pd = np.diag(np.linspace(1.0, 3.0, 40))
    prec = lambda v: np.linalg.solve(Pd, v)
    _, it, hist = gmres.gmres(lambda v: A @ v, b, prec, tol=1e-30, maxit=8)
    C = np.linalg.solve(Pd, A)
    z0 = prec(b)
    K = [z0]
    for k in range(1, 9):
        Kk = np.stack(K, axis=1)
        Kk = Kk / np.linalg.norm(Kk, axis=0)
        y = np.linalg.lstsq(C @ Kk, z0, rcond=None)[0]
        ref = np.linalg.norm(z0 - C @ Kk @ y) / np.linalg.norm(z0)
        assert abs(hist[k] - ref) < 1e-9 * max(ref, 1e-3), k
        K.append(C @ K[-1])


def test_gmres_equals_minres_on_symmetric_systems():
    """With P = I both minimize ||b - A x||_2 over the same Krylov space (symmetric indefinite A)."""
    rng = np.random.default_rng(3)
    Q, _ = np.linalg.qr(rng.standard_normal((300, 300)))
    A = Q @ np.diag(np.concatenate([-np.linspace(1, 2, 100), np.linspace(1, 2, 200)])) @ Q.T
    b = rng.standard_normal(300)
    _, itg, hg = gmres.gmres(lambda v: A @ v, b, lambda v: v, tol=1e-8)
    _, itm, hm = minres.minres(lambda v: A @ v, b, lambda v: v, tol=1e-8)
    assert itg == itm
    assert max(abs(a - c) / max(c, 1e-12) for a, c in zip(hg, hm)) < 1e-8


def _dense_blocks(D, disc, p, n_el, scaled):
    d = spaces.build(D, disc, p, n_el)
    op = stokes.StokesCube(D, disc, p, n_el)
    dv = dq = None
    if scaled:
        rng = np.random.default_rng(5)
        dv = rng.uniform(0.5, 1.5, sum(d.sizes[:-1]))
        dq = rng.uniform(0.5, 1.5, d.sizes[-1])
    PV = []
    o = d.offsets()
    for k, c in enumerate(d.comps):
        R = fd.assemble_R(c.Ks, c.Ms, c.coef)
        if dv is not None:
            s = np.sqrt(dv[o[k]:o[k + 1]])
            R = s[:, None] * R * s[None, :]
        PV.append(R)
    nv = int(o[-2])
    PVd = np.zeros((nv, nv))
    for k in range(D):
        PVd[o[k]:o[k + 1], o[k]:o[k + 1]] = PV[k]
    PQ = np.array([[1.0]])
    for M in d.Mq:                                 # M_D (x) .. (x) M_1, i1 fastest
        PQ = np.kron(M, PQ)
    if dq is not None:
        s = np.sqrt(dq)
        PQ = s[:, None] * PQ * s[None, :]
    B = np.zeros((op.sizes[-1], nv))
    for j in range(nv):
        e = np.zeros(nv)
        e[j] = 1.0
        B[:, j] = op.B_apply(e)
    return d, op, dv, dq, PVd, PQ, B


@pytest.mark.parametrize("D,disc,p,n_el,scaled", [(3, "TH", 2, 2, False), (2, "RT", 2, 3, True),
                                                  (3, "RT", 1, 2, True), (2, "TH", 3, 2, False)])
def test_triangular_and_constrained_vs_dense(D, disc, p, n_el, scaled):
    d, op, dv, dq, PV, PQ, B = _dense_blocks(D, disc, p, n_el, scaled)
    nv = PV.shape[0]
    nq = PQ.shape[0]
    PT = np.block([[PV, B.T], [np.zeros((nq, nv)), -PQ]])
    PC = np.block([[PV, B.T], [B, B @ np.linalg.solve(PV, B.T) - PQ]])
    blk = precond.BlockPrecond(d, dv, dq)
    r = np.random.default_rng(7).standard_normal(nv + nq)
    sT = precond.TriangularPrecond(blk, op).apply(r)
    sC = precond.ConstrainedPrecond(blk, op).apply(r)
    assert np.linalg.norm(sT - np.linalg.solve(PT, r)) < 1e-10 * np.linalg.norm(sT)
    assert np.linalg.norm(sC - np.linalg.solve(PC, r)) < 1e-9 * np.linalg.norm(sC)


def test_bt_is_transpose_of_b():
    op = stokes.StokesCube(3, "RT", 2, 2)
    rng = np.random.default_rng(9)
    u = rng.standard_normal(sum(op.sizes[:-1]))
    q = rng.standard_normal(op.sizes[-1])
    assert abs(q @ op.B_apply(u) - u @ op.BT_apply(q)) < 1e-13 * np.linalg.norm(u) * np.linalg.norm(q)


@pytest.mark.parametrize("D,disc,p,n_el", [(2, "TH", 2, 8), (3, "RT", 2, 3)])
def test_block_gmres_solves_stokes(D, disc, p, n_el):
    """P_T- and P_C-GMRES solve the (projected, consistent) Stokes system; their counts are below
    P_D-MINRES's, as in the paper's Tables 5-6 vs Table 3."""
    d = spaces.build(D, disc, p, n_el)
    op = stokes.StokesCube(D, disc, p, n_el)
    f = stokes.project_rhs(np.random.default_rng(0).standard_normal(op.n), op.sizes[-1])
    blk = precond.BlockPrecond(d)
    _, itd, _ = minres.minres(op.matvec, f, blk.apply)
    for P in (precond.TriangularPrecond(blk, op), precond.ConstrainedPrecond(blk, op)):
        x, it, _ = gmres.gmres(op.matvec, f, P.apply)
        x[-op.sizes[-1]:] -= x[-op.sizes[-1]:].mean()   # drop the null-space (constant p) part
        assert np.linalg.norm(op.matvec(x) - f) < 1e-5 * np.linalg.norm(f)  # preconditioned tol 1e-8
        assert it < itd, (type(P).__name__, it, itd)
