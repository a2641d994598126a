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


# Hand-evaluated Greville abscissae (xi_{j+1} + ... + xi_{j+deg}) / deg for RT p = 2 (alpha = 1),
# n_el = 2 (C-6, C-8):
#   own direction S^3_2, knots [0,0,0,0,1/2,1,1,1,1] -> [0, 1/6, 1/2, 5/6, 1], interior (first
#     and last dropped): [1/6, 1/2, 5/6];
#   tangential S^2_1 (full), knots [0,0,0,1/2,1,1,1] -> [0, 1/4, 3/4, 1];
#   pressure S^2_1 (full): [0, 1/4, 3/4, 1].
_G_OWN = [1 / 6, 1 / 2, 5 / 6]
_G_TAN = [0.0, 1 / 4, 3 / 4, 1.0]


def _nu_asym(x, y, z):
    """An axis-asymmetric coefficient: each direction carries a different weight, so a swapped
    Greville set, a kept boundary dof or a C-order reshape changes the sampled values."""
    return 1.0 + x + 10.0 * y + 100.0 * z


def test_nu_scalings_pinned_axis_asymmetric():
    """Config 3's D_V / D_Q sampling (C-6: D_V[i] = nu(Greville point of dof i), D_Q = 1/nu) on RT
    p = 2, n_el = 2 against hand-evaluated values at named dofs and against the full tensor grid
    typed out from the hand Greville lists (vec order i1 fastest)."""
    disc = spaces.build(3, "RT", 2, 2)
    assert [c.dims for c in disc.comps] == [[3, 4, 4], [4, 3, 4], [4, 4, 3]]
    dv, dq = spaces.nu_scalings(disc, _nu_asym)
    o = disc.offsets()
    # named dofs: component 1, (i1, i2, i3) = (1, 2, 3) -> (1/2, 3/4, 1): 1 + .5 + 7.5 + 100
    assert dv[o[0] + 1 + 3 * 2 + 12 * 3] == pytest.approx(109.0, rel=1e-15)
    # component 2, (3, 0, 1) -> (1, 1/6, 1/4): 1 + 1 + 10/6 + 25
    assert dv[o[1] + 3 + 4 * 0 + 12 * 1] == pytest.approx(1 + 1 + 10 / 6 + 25, rel=1e-15)
    # component 3, (1, 2, 2) -> (1/4, 3/4, 5/6): 1 + 1/4 + 7.5 + 500/6
    assert dv[o[2] + 1 + 4 * 2 + 16 * 2] == pytest.approx(1 + 0.25 + 7.5 + 500 / 6, rel=1e-15)
    # component 1's first dof sits at the first INTERIOR own-direction point: (1/6, 0, 0)
    assert dv[o[0]] == pytest.approx(1 + 1 / 6, rel=1e-15)
    # pressure (2, 1, 3) -> (3/4, 1/4, 1): 1/(1 + .75 + 2.5 + 100)
    assert dq[2 + 4 * 1 + 16 * 3] == pytest.approx(1 / 104.25, rel=1e-15)
    for k in range(3):
        g = [_G_OWN if d == k else _G_TAN for d in range(3)]
        exp = [_nu_asym(g[0][i1], g[1][i2], g[2][i3])
               for i3 in range(len(g[2])) for i2 in range(len(g[1])) for i1 in range(len(g[0]))]
        np.testing.assert_allclose(dv[o[k]:o[k + 1]], exp, rtol=1e-15)
    expq = [1 / _nu_asym(_G_TAN[i1], _G_TAN[i2], _G_TAN[i3])
            for i3 in range(4) for i2 in range(4) for i1 in range(4)]
    np.testing.assert_allclose(dq, expq, rtol=1e-15)
