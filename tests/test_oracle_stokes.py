"""Pins for the MINRES harness (oracle/stokes.py, oracle/minres.py): the Kronecker Stokes
operator against brute-force 3D quadrature of a(.,.) and b(.,.), its
symmetry and null space, Theorem 1's spectral bounds on the cube, and MINRES against a dense
solve."""
import itertools

import numpy as np
import pytest

from oracle import fd, minres, precond, spaces, splines, stokes
import test_oracle_assembly as asm


def _dense(op):
    n = op.n
    A = np.zeros((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        A[:, j] = op.matvec(e)
    return A


@pytest.mark.parametrize("disc,p,n_el", [("TH", 1, 2), ("RT", 2, 2)])
def test_operator_symmetric_and_null_space(disc, p, n_el):
    op = stokes.StokesCube(3, disc, p, n_el)
    A = _dense(op)
    assert np.max(np.abs(A - A.T)) < 1e-13 * np.max(np.abs(A))
    # (0, 1_p) spans the null space: B_r^T 1 = 0 (partition of unity + boundary restriction)
    z = np.zeros(op.n)
    z[op.off_idx[3]:] = 1.0
    assert np.max(np.abs(A @ z)) < 1e-13
    # the pressure-pressure block is zero
    assert np.all(A[op.off_idx[3]:, op.off_idx[3]:] == 0.0)


@pytest.mark.parametrize("disc,p,n_el,own", [("TH", 1, 2, None), ("RT", 2, 2, None), ("TH", 2, 1, None),
                                              ("RT", 2, 2, 1)])
def test_diagonal_blocks_equal_pv(disc, p, n_el, own):
    # A_kk = P_V,k on the identity map; own = 1: the literal C-3 reading
    op = stokes.StokesCube(3, disc, p, n_el, rt_own_alpha=own)
    A = _dense(op)
    d = spaces.build(3, disc, p, n_el, rt_own_alpha=own)
    o = op.off_idx
    for k, c in enumerate(d.comps):
        R = fd.assemble_R(c.Ks, c.Ms, c.coef)
        blk = A[o[k]:o[k + 1], o[k]:o[k + 1]]
        assert np.max(np.abs(blk - R)) < 1e-12 * np.max(np.abs(R))


def _brute_velocity_pressure(p, n_el, nu=None, q=None):
    """TH velocity block and B by direct 3D quadrature of a(.,.) and b(.,.),
    a(w, v) = int 2 nu grad^s w : grad^s v."""
    spV = [asm._space(p + 1, p - 1, n_el, True)] * 3
    spQ = [asm._space(p, p - 1, n_el, False)] * 3
    X, W = asm._grid([n_el] * 3, q or p + 3)
    Wnu = W if nu is None else W * nu(X[:, 0], X[:, 1], X[:, 2])
    _, GV, nv = asm._trivariate(spV, X)
    BQ, _, nq = asm._trivariate(spQ, X)
    Nv = GV.shape[1]
    E = np.eye(3)
    A = np.zeros((3 * Nv, 3 * Nv))
    for r, s in itertools.product(range(3), range(3)):
        blk = np.zeros((Nv, Nv))
        for q in range(len(W)):
            gi = np.einsum("a,ib->iab", E[r], GV[q])   # grad(e_r phi_i)
            gj = np.einsum("a,jb->jab", E[s], GV[q])
            si = 0.5 * (gi + gi.transpose(0, 2, 1))
            sj = 0.5 * (gj + gj.transpose(0, 2, 1))
            blk += Wnu[q] * 2.0 * np.einsum("iab,jab->ij", si, sj)
        A[r * Nv:(r + 1) * Nv, s * Nv:(s + 1) * Nv] = blk
    B = np.zeros((BQ.shape[1], 3 * Nv))
    for r in range(3):
        # b(phi_j^r, rho_l) = -int rho_l d_r phi_j
        B[:, r * Nv:(r + 1) * Nv] = -np.einsum("q,ql,qj->lj", W, BQ, GV[:, :, r])
    return A, B


def test_th_operator_matches_brute_force_quadrature():
    p, n_el = 1, 2
    op = stokes.StokesCube(3, "TH", p, n_el)
    A = _dense(op)
    Ab, Bb = _brute_velocity_pressure(p, n_el)
    nv = op.off_idx[3]
    assert np.max(np.abs(A[:nv, :nv] - Ab)) < 1e-13 * np.max(np.abs(Ab))
    assert np.max(np.abs(A[nv:, :nv] - Bb)) < 1e-13 * np.max(np.abs(Bb))
    assert np.max(np.abs(A[:nv, nv:] - Bb.T)) < 1e-13 * np.max(np.abs(Bb))


def test_variable_viscosity_operator_matches_brute_force():
    """Config 3's nu = 1 + 0.5 sin sin sin as two separable Kronecker terms (synth.viscosity)."""
    import synth
    p, n_el = 1, 2
    op = stokes.StokesCube(3, "TH", p, n_el, nu_terms=stokes.config3_nu_terms())
    A = _dense(op)
    Ab, Bb = _brute_velocity_pressure(p, n_el, nu=synth.viscosity, q=p + 7)
    nv = op.off_idx[3]
    assert np.max(np.abs(A[:nv, :nv] - Ab)) < 1e-13 * np.max(np.abs(Ab))
    assert np.max(np.abs(A[nv:, :nv] - Bb)) < 1e-13 * np.max(np.abs(Bb))


@pytest.mark.parametrize("disc,p,n_el", [("TH", 1, 2), ("TH", 2, 2), ("RT", 2, 2)])
def test_theorem1_bounds_on_cube(disc, p, n_el):
    # eig(P_V^{-1} A) in [delta, Delta] = [1/2, 2] for the identity map (Theorem 1)
    op = stokes.StokesCube(3, disc, p, n_el)
    A = _dense(op)
    nv = op.off_idx[3]
    Av = A[:nv, :nv]
    d = spaces.build(3, disc, p, n_el)
    PV = np.zeros_like(Av)
    o = op.off_idx
    for k, c in enumerate(d.comps):
        PV[o[k]:o[k + 1], o[k]:o[k + 1]] = fd.assemble_R(c.Ks, c.Ms, c.coef)
    import scipy.linalg
    ev = scipy.linalg.eigh(Av, PV, eigvals_only=True)
    assert ev.min() >= 0.5 - 1e-10 and ev.max() <= 2.0 + 1e-10


def test_minres_matches_dense_solve():
    op = stokes.StokesCube(3, "TH", 1, 2)
    A = _dense(op)
    d = spaces.build(3, "TH", 1, 2)
    P = precond.BlockPrecond(d)
    f = stokes.project_rhs(np.random.default_rng(0).standard_normal(op.n), op.sizes[-1])
    x, its, hist = minres.minres(op.matvec, f, P.apply, tol=1e-12)
    assert np.linalg.norm(A @ x - f) / np.linalg.norm(f) < 1e-9
    # minimum-norm solution of the consistent singular system equals lstsq's up to the null space
    xl = np.linalg.lstsq(A, f, rcond=None)[0]
    dx = x - xl
    dx[op.off_idx[3]:] -= dx[op.off_idx[3]:].mean()
    assert np.linalg.norm(dx) / np.linalg.norm(xl) < 1e-8
    assert all(b <= a * (1 + 1e-12) for a, b in zip(hist, hist[1:]))  # monotone (MINRES)
    assert its <= op.n


def test_minres_finite_termination_spd():
    rng = np.random.default_rng(1)
    Q, _ = np.linalg.qr(rng.standard_normal((12, 12)))
    A = Q @ np.diag(np.linspace(1.0, 10.0, 12)) @ Q.T   # 12 distinct eigenvalues
    b = rng.standard_normal(12)
    x, its, _ = minres.minres(lambda v: A @ v, b, lambda r: r, tol=1e-13)
    assert its <= 12
    assert np.allclose(A @ x, b, atol=1e-10)


def test_paper_scalings_constant_viscosity_closed_form():
    """nu == c (constant): A_kk = c P_V,k and Q = P_Q / c, so D_V == c and D_Q == 1/c."""
    d = spaces.build(3, "RT", 2, 3)
    c = 1.7
    op = stokes.StokesCube(3, "RT", 2, 3, nu_terms=[(c, None)])
    dv, dq = stokes.nu_scalings_paper(d, op, lambda x, y, z: c + 0.0 * x, q=6)
    assert np.max(np.abs(dv - c)) < 1e-12 * c
    assert np.max(np.abs(dq - 1.0 / c)) < 1e-12


def test_paper_pressure_diagonal_brute_force():
    """diag(Q), Q = int nu^{-1} rho_i rho_j, by three tensor contractions = the diagonal of the
    densely assembled 3D quadrature (tiny grid, config 3's viscosity)."""
    import synth
    p, n_el, q = 2, 2, 6
    d = spaces.build(3, "RT", p, n_el)
    op = stokes.StokesCube(3, "RT", p, n_el)
    _, dq = stokes.nu_scalings_paper(d, op, synth.viscosity, q)
    spQ = [asm._space(p, p - 1, n_el, False)] * 3
    X, W = asm._grid([n_el] * 3, q)
    BQ, _, _ = asm._trivariate(spQ, X)
    wn = W / synth.viscosity(X[:, 0], X[:, 1], X[:, 2])
    diagQ = np.einsum("q,qi->i", wn, BQ ** 2)
    PQ = np.kron(d.Mq[2], np.kron(d.Mq[1], d.Mq[0]))
    assert np.max(np.abs(dq * np.diag(PQ) - diagQ)) < 1e-13 * np.max(diagQ)


def test_paper_velocity_scaling_is_operator_diagonal_ratio():
    """D_V diag(P_V,k) = diag(A_kk) of the densely applied nu-weighted operator (tiny RT grid)."""
    p, n_el = 1, 2
    d = spaces.build(3, "RT", p, n_el)
    op = stokes.StokesCube(3, "RT", p, n_el, nu_terms=stokes.config3_nu_terms(3))
    import synth
    dv, _ = stokes.nu_scalings_paper(d, op, synth.viscosity, q=6)
    A = _dense(op)
    o = op.off_idx
    for k, c in enumerate(d.comps):
        R = fd.assemble_R(c.Ks, c.Ms, c.coef)
        blk = np.diag(A[o[k]:o[k + 1], o[k]:o[k + 1]])
        assert np.max(np.abs(dv[o[k]:o[k + 1]] * np.diag(R) - blk)) < 1e-12 * np.max(np.abs(blk))
