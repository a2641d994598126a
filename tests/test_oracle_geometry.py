"""Pins for the NEXT-3 oracle (oracle/geometry.py): the annulus map against
its closed-form values and a complex-step Jacobian, the mapped TH Stokes operator against
brute-force 3D quadrature of the weak form in physical coordinates with a
numerically inverted Jacobian, the identity-geometry collapse to the cube, the separable fit on
exactly separable data, and the diagonal scalings of §6."""
import itertools
import math

import numpy as np
import pytest

from oracle import fd, geometry, minres, precond, spaces, splines, stokes
import test_oracle_assembly as asm


def _cs_jacobian(G, e):
    """J[a, b] = dG_a / d eta_b by complex step (exact to rounding, independent of the Sep J^{-1})."""
    h = 1e-30
    J = np.zeros((3, 3))
    for b in range(3):
        ee = [complex(v) for v in e]
        ee[b] += 1j * h
        J[:, b] = np.imag(G(*[np.array(v) for v in ee])) / h
    return J


def test_annulus_closed_form_values():
    geo = geometry.annulus()
    assert np.allclose(geo.G(0.0, 0.0, 0.0), [1.0, 0.0, 0.0], atol=1e-15)
    assert np.allclose(geo.G(1.0, 1.0, 0.5), [math.sqrt(2), math.sqrt(2), 0.5], atol=1e-15)
    assert abs(geo.detJ(0.0, 0.0, 0.0) - math.pi / 4) < 1e-15
    assert abs(geo.detJ(1.0, 0.3, 0.7) - math.pi / 2) < 1e-15
    rng = np.random.default_rng(0)
    for e in rng.uniform(0, 1, (5, 3)):
        J = _cs_jacobian(geo.G, e)
        Ji = np.array([[geo.Jinv[a][b](*e) for b in range(3)] for a in range(3)], dtype=float)
        assert np.max(np.abs(Ji - np.linalg.inv(J))) < 1e-14
        assert abs(geo.detJ(*e) - abs(np.linalg.det(J))) < 1e-14


def test_identity_coefficients():
    geo = geometry.identity(3)
    for r, s in itertools.product(range(3), range(3)):
        C = geometry.coefficient(geo, r, s)
        M = np.array([[float(C[d][e](0.3, 0.4, 0.5)) for e in range(3)] for d in range(3)])
        ref = (np.eye(3) if r == s else 0.0) + np.outer(np.eye(3)[s], np.eye(3)[r])
        assert np.array_equal(M, ref)


def _brute(geo, p, n_el, q):
    """A (velocity block) and B by 3D quadrature of int 2 grad^s u : grad^s v dx and
    -int q div v dx in physical coordinates: grad_x phi = J^{-T} grad_eta phi, dx = |det J| deta."""
    spV = [asm._space(p + 1, p - 1, n_el, True)] * 3
    spQ = [asm._space(p, p - 1, n_el, False)] * 3
    X, W = asm._grid([n_el] * 3, q)
    _, GV, _ = asm._trivariate(spV, X)
    BQ, _, _ = asm._trivariate(spQ, X)
    Nv, Nq = GV.shape[1], BQ.shape[1]
    Gx = np.zeros_like(GV)
    wdet = np.zeros(len(X))
    for i, e in enumerate(X):
        J = _cs_jacobian(geo.G, e)
        Gx[i] = np.linalg.solve(J.T, GV[i].T).T          # J^{-T} grad_eta
        wdet[i] = W[i] * abs(np.linalg.det(J))
    A = np.zeros((3 * Nv, 3 * Nv))
    B = np.zeros((Nq, 3 * Nv))
    for r in range(3):
        for s in range(3):
            # u = e_s phi_j, v = e_r phi_i: 2 grad^s u : grad^s v = delta_rs grad phi_i . grad phi_j
            #   + d_{x_s} phi_i d_{x_r} phi_j
            blk = np.einsum("q,qi,qj->ij", wdet, Gx[:, :, s], Gx[:, :, r])
            if r == s:
                blk = blk + np.einsum("q,qid,qjd->ij", wdet, Gx, Gx)
            A[r * Nv:(r + 1) * Nv, s * Nv:(s + 1) * Nv] = blk
        B[:, r * Nv:(r + 1) * Nv] = -np.einsum("q,ql,qj->lj", wdet, BQ, Gx[:, :, r])
    return A, B


def _dense(op):
    A = np.zeros((op.n, op.n))
    for j in range(op.n):
        e = np.zeros(op.n)
        e[j] = 1.0
        A[:, j] = op.matvec(e)
    return A


@pytest.mark.parametrize("p,n_el", [(1, 2), (2, 1)])
def test_mapped_operator_matches_brute_force(p, n_el):
    geo = geometry.annulus()
    op = geometry.StokesMapped(geo, p, n_el)
    Ad = _dense(op)
    A, B = _brute(geo, p, n_el, op.q)
    nv = 3 * op.sizes[0]
    sc = np.max(np.abs(A))
    assert np.max(np.abs(Ad[:nv, :nv] - A)) < 1e-12 * sc
    assert np.max(np.abs(Ad[nv:, :nv] - B)) < 1e-12 * sc
    assert np.max(np.abs(Ad - Ad.T)) < 1e-12 * sc
    assert np.all(Ad[nv:, nv:] == 0.0)
    # constant pressure is in the null space (divergence theorem, zero-trace velocities) up to
    # the Gauss rule's error on the trigonometric metric terms
    z = np.zeros(op.n)
    z[nv:] = 1.0
    assert np.max(np.abs(Ad @ z)) < 1e-9 * sc


def test_identity_geometry_is_the_cube():
    op = geometry.StokesMapped(geometry.identity(3), 2, 2, q=5)
    cube = stokes.StokesCube(3, "TH", 2, 2)
    x = np.random.default_rng(1).standard_normal(op.n)
    assert np.linalg.norm(op.matvec(x) - cube.matvec(x)) < 1e-12 * np.linalg.norm(cube.matvec(x))


def test_separable_fit_exact_products():
    rng = np.random.default_rng(2)
    n = (7, 5, 6)
    tb = [np.exp(rng.uniform(-1, 1, n[d])) for d in range(3)]
    mb = [np.exp(rng.uniform(-1, 1, n[d])) for d in range(3)]
    E = np.meshgrid(*[np.arange(k) for k in n], indexing="ij")
    c = []
    for d in range(3):
        v = tb[d][E[d]]
        for m in range(3):
            if m != d:
                v = v * mb[m][E[m]]
        c.append(v)
    tau, mu, hist = geometry.separable_fit(c, tol=1e-15, max_sweeps=200)
    for d in range(3):
        v = tau[d][E[d]]
        for m in range(3):
            if m != d:
                v = v * mu[m][E[m]]
        assert np.max(np.abs(v / c[d] - 1)) < 1e-8
    for m in range(3):
        assert abs(np.log(mu[m]).mean()) < 1e-12      # gauge
    assert all(b <= a * (1 + 1e-9) + 1e-24 * hist[0] for a, b in zip(hist, hist[1:]))  # monotone descent


def test_separable_fit_identity_and_constants():
    x, _ = geometry.quadrature_grid(3, 4)
    for k in range(3):
        c = geometry.sample_diagonal(geometry.identity(3), k, x)
        tau, mu, _ = geometry.separable_fit(c)
        for d in range(3):
            assert np.allclose(tau[d], 2.0 if d == k else 1.0, rtol=1e-14)
            assert np.allclose(mu[d], 1.0, rtol=1e-14)


def test_identity_geo_pencils_reproduce_plain_pv():
    p, n_el = 2, 3
    op = geometry.StokesMapped(geometry.identity(3), p, n_el)
    disc, dv, dq = geometry.geo_discretization(op)
    plain = spaces.build(3, "TH", p, n_el)
    for k in range(3):
        Rg = fd.assemble_R(disc.comps[k].Ks, disc.comps[k].Ms, disc.comps[k].coef)
        Rp = fd.assemble_R(plain.comps[k].Ks, plain.comps[k].Ms, plain.comps[k].coef)
        assert np.max(np.abs(Rg - Rp)) < 1e-12 * np.max(np.abs(Rp))
    assert np.allclose(dv, 1.0, rtol=1e-12) and np.allclose(dq, 1.0, rtol=1e-12)


def test_annulus_diagonals_and_scalings():
    """diag(A_kk) from the Kronecker diagonals equals the assembled block's diagonal;
    D_V diag(P^_V) = diag(A), D_Q diag(P_Q) = diag(Q) with Q by brute-force quadrature."""
    p, n_el = 1, 2
    geo = geometry.annulus()
    op = geometry.StokesMapped(geo, p, n_el)
    Ad = _dense(op)
    disc, dv, dq = geometry.geo_discretization(op)
    o = op.off_idx
    for k in range(3):
        blk = np.diag(Ad[o[k]:o[k + 1], o[k]:o[k + 1]])
        assert np.max(np.abs(op.diag_A(k) - blk)) < 1e-13 * np.max(blk)
        c = disc.comps[k]
        R = fd.assemble_R(c.Ks, c.Ms, c.coef)
        assert np.max(np.abs(dv[o[k]:o[k + 1]] * np.diag(R) - blk)) < 1e-12 * np.max(blk)
    spQ = [asm._space(p, p - 1, n_el, False)] * 3
    X, W = asm._grid([n_el] * 3, op.q)
    BQ, _, _ = asm._trivariate(spQ, X)
    wdet = W * np.array([abs(np.linalg.det(_cs_jacobian(geo.G, e))) for e in X])
    Qd = np.einsum("q,qi->i", wdet, BQ ** 2)
    Mq = disc.Mq[0]
    PQd = np.kron(np.diag(Mq), np.kron(np.diag(Mq), np.diag(Mq)))
    assert np.max(np.abs(dq * PQd - Qd)) < 1e-13 * np.max(Qd)


def test_geometry_aware_preconditioner_reduces_minres_iterations():
    """on the annulus the geometry-aware P_D^G needs far fewer MINRES iterations
    than the plain P_D (the paper: about half)."""
    op = geometry.StokesMapped(geometry.annulus(), 2, 4)
    f = stokes.project_rhs(np.random.default_rng(0).standard_normal(op.n), op.sizes[-1])
    _, it_plain, _ = minres.minres(op.matvec, f, precond.BlockPrecond(geometry.plain_discretization(op)).apply)
    disc, dv, dq = geometry.geo_discretization(op)
    _, it_geo, _ = minres.minres(op.matvec, f, precond.BlockPrecond(disc, dv, dq).apply)
    assert it_geo < 0.8 * it_plain, (it_geo, it_plain)


def test_mapped_b_and_bt_consistent_with_matvec():
    op = geometry.StokesMapped(geometry.annulus(), 1, 2)
    rng = np.random.default_rng(4)
    nv = int(op.off_idx[-2])
    u = rng.standard_normal(nv)
    q = rng.standard_normal(op.sizes[-1])
    x = np.concatenate([u, np.zeros(op.sizes[-1])])
    assert np.allclose(op.matvec(x)[nv:], op.B_apply(u), rtol=0, atol=1e-14)
    x = np.concatenate([np.zeros(nv), q])
    assert np.allclose(op.matvec(x)[:nv], op.BT_apply(q), rtol=0, atol=1e-14)
