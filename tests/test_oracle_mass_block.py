"""Pins for oracle/mass.py and oracle/precond.py."""
import numpy as np
import pytest
import scipy.linalg

from oracle import fd, kron, mass, precond, spaces, univariate
import synth


def test_kron_matvec_matches_dense():
    rng = np.random.default_rng(0)
    A = [rng.standard_normal((n, n)) for n in (3, 4, 2)]   # A_3, A_2, A_1 (slowest first)
    x = rng.standard_normal(24)
    assert np.allclose(kron.kron_matvec(A, x), kron.kron_dense(A) @ x, rtol=1e-14, atol=1e-14)


def test_kron_scalar_and_identity():
    assert kron.kron_matvec([np.array([[2.0]]), np.array([[3.0]]), np.array([[4.0]])], np.ones(1))[0] == 24.0
    x = np.arange(6.0)
    assert np.array_equal(kron.kron_matvec([np.eye(2), np.eye(3)], x), x)


@pytest.mark.parametrize("p,n_el", [(2, 3), (3, 4), (5, 2)])
def test_mass_inverse_dense_and_round_trip(p, n_el):
    M = univariate.pressure_mass(p, n_el)
    Ms = [M, univariate.pressure_mass(p, n_el + 1), univariate.pressure_mass(p, n_el + 2)]
    km = mass.KronMass(Ms)
    assert km.bands == [p, p, p]
    t = np.random.default_rng(p).standard_normal(int(np.prod(km.dims)))
    x = km.inverse(t)
    dense = kron.kron_dense(list(reversed(Ms)))
    kappa = np.linalg.cond(dense)
    # forward error of two backward-stable solves is O(kappa eps)
    assert np.linalg.norm(x - scipy.linalg.solve(dense, t)) / np.linalg.norm(x) < 50 * kappa * 2.2e-16
    assert np.linalg.norm(km.forward(x) - t) / np.linalg.norm(t) < 50 * kappa * 2.2e-16


def test_mass_diagonal_factors():
    Ms = [np.diag([1.0, 2.0]), np.diag([3.0])]
    km = mass.KronMass(Ms)
    assert np.allclose(km.inverse(np.array([6.0, 6.0])), [2.0, 1.0])


def test_mass_constant_scaling():
    M = univariate.pressure_mass(3, 3)
    km = mass.KronMass([M, M, M])
    t = np.random.default_rng(9).standard_normal(M.shape[0] ** 3)
    assert np.allclose(km.scaled_inverse(t, np.full(t.shape, 5.0)), km.inverse(t) / 5.0, rtol=1e-14)


def test_block_equals_pieces_and_spd():
    disc = spaces.build(3, "RT", 2, 2)
    P = precond.BlockPrecond(disc)
    r = np.random.default_rng(11).standard_normal(disc.n_total)
    s = P.apply(r)
    o = disc.offsets()
    for k, c in enumerate(disc.comps):
        xd = fd.dense_solve(c.Ks, c.Ms, c.coef, r[o[k]:o[k + 1]])
        assert np.linalg.norm(s[o[k]:o[k + 1]] - xd) / np.linalg.norm(xd) < 1e-12
    PQ = kron.kron_dense(list(reversed(disc.Mq)))
    xq = np.linalg.solve(PQ, r[o[3]:])
    assert np.linalg.norm(s[o[3]:] - xq) / np.linalg.norm(xq) < 1e-12
    assert r @ s > 0
    # batch semantics: rows independent (C-14)
    R2 = np.stack([r, 2 * r])
    S2 = P.apply(R2)
    assert np.allclose(S2[0], s) and np.allclose(S2[1], 2 * s)


def test_block_2d_th():
    disc = spaces.build(2, "TH", 2, 3)
    P = precond.BlockPrecond(disc)
    r = np.random.default_rng(12).standard_normal(disc.n_total)
    s = P.apply(r)
    o = disc.offsets()
    for k, c in enumerate(disc.comps):
        assert c.coef == [1.0 + (d == k) for d in range(2)]
        xd = fd.dense_solve(c.Ks, c.Ms, c.coef, r[o[k]:o[k + 1]])
        assert np.linalg.norm(s[o[k]:o[k + 1]] - xd) / np.linalg.norm(xd) < 1e-12


def test_scaled_block_dense():
    disc = spaces.build(3, "TH", 1, 3)
    dv, dq = spaces.nu_scalings(disc, synth.viscosity)
    assert dv.shape == (sum(disc.sizes[:3]),) and dq.shape == (disc.sizes[3],)
    assert dv.min() >= 0.5 and dv.max() <= 1.5
    P = precond.BlockPrecond(disc, dv, dq)
    r = np.random.default_rng(13).standard_normal(disc.n_total)
    s = P.apply(r)
    o = disc.offsets()
    for k, c in enumerate(disc.comps):
        Dk = dv[o[k]:o[k + 1]]
        R = fd.assemble_R(c.Ks, c.Ms, c.coef)
        PG = np.sqrt(Dk)[:, None] * R * np.sqrt(Dk)[None, :]   # D^{1/2} P D^{1/2}
        xd = np.linalg.solve(PG, r[o[k]:o[k + 1]])
        assert np.linalg.norm(s[o[k]:o[k + 1]] - xd) / np.linalg.norm(xd) < 1e-12
        # diag(D^{1/2} P D^{1/2}) = D diag(P) (P:1059 definition of D as a ratio)
        assert np.allclose(np.diag(PG), Dk * np.diag(R), rtol=1e-14)


def test_greville_scaling_constant_nu():
    disc = spaces.build(3, "RT", 2, 2)
    dv, dq = spaces.nu_scalings(disc, lambda x, y, z: 3.0 + 0 * x)
    assert np.allclose(dv, 3.0) and np.allclose(dq, 1.0 / 3.0)
