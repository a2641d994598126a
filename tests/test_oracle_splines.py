"""Pins for oracle/splines.py against closed forms and invariants."""
import json
import math
import os

import numpy as np
import pytest

from oracle import splines, spaces

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("q", [1, 2, 3, 5, 8])
def test_gauss_legendre_exact_monomials(q):
    x, w = splines.gauss_legendre(q)
    for k in range(2 * q):
        assert abs(np.sum(w * x**k) - 1.0 / (k + 1)) < 1e-14


def test_gauss_legendre_small_rules():
    x, w = splines.gauss_legendre(1)
    assert np.allclose(x, [0.5]) and np.allclose(w, [1.0])
    x, w = splines.gauss_legendre(2)
    assert np.allclose(np.sort(x), [0.5 - 1 / (2 * math.sqrt(3)), 0.5 + 1 / (2 * math.sqrt(3))], atol=1e-15)
    assert np.allclose(w, [0.5, 0.5])


@pytest.mark.parametrize("p,alpha,n_el,m", [(1, 0, 1, 2), (2, 1, 2, 4), (3, 2, 4, 7), (4, 3, 64, 68),
                                             (5, 4, 64, 69), (6, 4, 128, 261), (2, 0, 3, 7)])
def test_dimension_formula(p, alpha, n_el, m):
    # m = n_el (p - alpha) + alpha + 1 (follows from P:176-199)
    assert splines.dimension(p, alpha, n_el) == m == n_el * (p - alpha) + alpha + 1


def test_knots_examples():
    assert np.allclose(splines.open_uniform_knots(1, 0, 1), [0, 0, 1, 1])
    assert np.allclose(splines.open_uniform_knots(2, 1, 2), [0, 0, 0, 0.5, 1, 1, 1])


@pytest.mark.parametrize("p,alpha,n_el", [(1, 0, 3), (2, 1, 4), (3, 2, 5), (4, 3, 3), (5, 2, 2), (6, 4, 4)])
def test_partition_of_unity_nonneg_endpoints(p, alpha, n_el):
    xi = splines.open_uniform_knots(p, alpha, n_el)
    eta = np.concatenate([[0.0, 1.0], np.random.default_rng(7).random(1000), np.unique(xi)])
    B = splines.basis(xi, p, eta)
    assert np.max(np.abs(B.sum(axis=1) - 1.0)) < 1e-13
    assert B.min() >= -1e-15
    # open knots interpolate at the ends: b_1(0) = b_m(1) = 1
    B01 = splines.basis(xi, p, [0.0, 1.0])
    assert B01[0, 0] == pytest.approx(1.0) and B01[1, -1] == pytest.approx(1.0)
    # support locality: at most p+1 non-zero functions at any point
    assert np.max(np.sum(B > 0, axis=1)) <= p + 1


def test_hat_functions_p1():
    xi = splines.open_uniform_knots(1, 0, 1)
    assert np.allclose(splines.basis(xi, 1, [0.25])[0], [0.75, 0.25])


@pytest.mark.parametrize("p", [1, 2, 3, 4, 6])
def test_single_element_is_bernstein(p):
    xi = splines.open_uniform_knots(p, p - 1, 1)
    eta = np.linspace(0, 1, 17)
    B = splines.basis(xi, p, eta)
    for i in range(p + 1):
        bern = math.comb(p, i) * eta**i * (1 - eta) ** (p - i)
        assert np.max(np.abs(B[:, i] - bern)) < 1e-14


@pytest.mark.parametrize("p,alpha,n_el", [(2, 1, 3), (3, 2, 4), (4, 3, 3), (5, 3, 2)])
def test_derivative_vs_central_difference(p, alpha, n_el):
    xi = splines.open_uniform_knots(p, alpha, n_el)
    # points away from breakpoints
    eta = (np.arange(n_el) + 0.37) / n_el
    hstep = 1e-6
    fd = (splines.basis(xi, p, eta + hstep) - splines.basis(xi, p, eta - hstep)) / (2 * hstep)
    d = splines.basis_derivative(xi, p, eta)
    assert np.max(np.abs(fd - d)) <= 1e-5 * max(1.0, np.max(np.abs(d)))
    # derivatives of a partition of unity sum to zero
    assert np.max(np.abs(d.sum(axis=1))) < 1e-10


def test_greville_reproduces_identity():
    # sum_j g_j b_j(eta) = eta (linear precision of the Greville abscissae)
    for p, a, n in [(2, 1, 4), (4, 3, 5), (5, 4, 3)]:
        xi = splines.open_uniform_knots(p, a, n)
        eta = np.linspace(0, 1, 31)
        assert np.max(np.abs(splines.basis(xi, p, eta) @ splines.greville(xi, p) - eta)) < 1e-14


def test_config_sizes_golden():
    """Space dimensions of BASELINE.json's configs (tests/golden/config_sizes.json: P:276, 296, 348)."""
    with open(os.path.join(GOLDEN, "config_sizes.json")) as f:
        gold = json.load(f)
    for key, g in gold["configs"].items():
        d = spaces.build(g["D"], g["disc"], g["p"], g["n_el"]) if g["n_el"] <= 64 else None
        if d is None:
            # large configs: check the 1D dimensions only (matrices would be slow to build here)
            a = g["p"] - 1
            if g["disc"] == "TH":
                n = splines.dimension(g["p"] + 1, a, g["n_el"]) - 2
                vel = [[n] * g["D"]] * g["D"]
            else:
                nn = splines.dimension(g["p"] + 1, a + 1, g["n_el"]) - 2
                nt = splines.dimension(g["p"], a, g["n_el"])
                vel = [[nn if dd == k else nt for dd in range(g["D"])] for k in range(g["D"])]
            q = [splines.dimension(g["p"], a, g["n_el"])] * g["D"]
        else:
            vel = [c.dims for c in d.comps]
            q = d.q_dims
        assert vel == g["velocity_dims"], key
        assert q == g["pressure_dims"], key
        tot = sum(int(np.prod(v)) for v in vel) + int(np.prod(q))
        assert tot == g["n_total"], key
