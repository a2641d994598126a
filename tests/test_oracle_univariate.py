"""Pins for oracle/univariate.py (M, K, K~ closed forms and invariants)."""
import numpy as np
import pytest

from oracle import splines, univariate


@pytest.mark.parametrize("p,alpha,n_el", [(1, 0, 5), (2, 1, 4), (3, 2, 6), (4, 3, 6), (5, 4, 3), (4, 2, 3)])
def test_full_mass_row_sums_and_total(p, alpha, n_el):
    K, M = univariate.stiffness_mass(p, alpha, n_el)
    xi = splines.open_uniform_knots(p, alpha, n_el)
    m = M.shape[0]
    # sum_s int b_l b_s = int b_l = (xi_{l+p+1} - xi_l)/(p+1)   (partition of unity)
    expect = np.array([(xi[l + p + 1] - xi[l]) / (p + 1) for l in range(m)])
    assert np.max(np.abs(M.sum(axis=1) - expect)) < 1e-15 * 10
    assert abs(M.sum() - 1.0) < 1e-14
    # K annihilates constants
    assert np.max(np.abs(K.sum(axis=1))) < 1e-12 * np.max(np.abs(K))
    assert np.allclose(M, M.T, atol=0, rtol=0) or np.max(np.abs(M - M.T)) < 1e-17
    assert np.max(np.abs(K - K.T)) <= 1e-15 * np.max(np.abs(K))


@pytest.mark.parametrize("p,alpha,n_el", [(2, 1, 6), (3, 2, 6), (5, 4, 8), (3, 0, 4)])
def test_bandwidth_is_degree(p, alpha, n_el):
    K, M = univariate.stiffness_mass(p, alpha, n_el)
    n = M.shape[0]
    for A in (K, M):
        for b in range(p + 1, n):
            assert np.all(np.diagonal(A, b) == 0.0)
    assert np.any(np.diagonal(M, p) != 0.0)


def test_p1_closed_forms():
    n_el = 7
    h = 1.0 / n_el
    K, M = univariate.stiffness_mass(1, 0, n_el)
    n = n_el + 1
    Me = (h / 6) * (np.diag(4 * np.ones(n)) + np.diag(np.ones(n - 1), 1) + np.diag(np.ones(n - 1), -1))
    Me[0, 0] = Me[-1, -1] = h / 3
    Ke = (1 / h) * (np.diag(2 * np.ones(n)) - np.diag(np.ones(n - 1), 1) - np.diag(np.ones(n - 1), -1))
    Ke[0, 0] = Ke[-1, -1] = 1 / h
    assert np.max(np.abs(M - Me)) < 1e-15
    assert np.max(np.abs(K - Ke)) < 1e-12


@pytest.mark.parametrize("cpen", [1.0, 3.0, 20.0])
def test_nitsche_p1_one_element(cpen):
    # P:701-704 with p = 1, one element, h = 1: K~ = [[2g-1, 1], [1, 2g-1]], g = C_pen/h
    Kt = univariate.nitsche_stiffness(1, 0, 1, cpen)
    g = cpen
    assert np.allclose(Kt, [[2 * g - 1, 1.0], [1.0, 2 * g - 1]], atol=1e-14)


@pytest.mark.parametrize("p,n_el", [(2, 4), (4, 8), (4, 64)])
def test_nitsche_symmetric_spd(p, n_el):
    Kt = univariate.nitsche_stiffness(p, p - 1, n_el, univariate.c_pen(p))
    assert np.max(np.abs(Kt - Kt.T)) < 1e-12 * np.max(np.abs(Kt))
    assert np.linalg.eigvalsh(Kt).min() > 0


def test_interior_restriction_sizes():
    K, M = univariate.th_velocity_pencil(3, 32)
    assert K.shape == M.shape == (65, 65)
    K, M = univariate.rt_normal_pencil(4, 64)
    assert K.shape == (67, 67)
    K, M = univariate.rt_tangential_pencil(4, 64)
    assert K.shape == (68, 68)
    assert univariate.pressure_mass(5, 128).shape == (133, 133)


def test_c_pen():
    assert univariate.c_pen(4) == 20.0  # 5 (alpha + 1), alpha = p - 1
