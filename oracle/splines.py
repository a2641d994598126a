"""Univariate B-splines (§2.1). Oracle: test infrastructure only."""
from __future__ import annotations

import numpy as np


def open_uniform_knots(p: int, alpha: int, n_el: int) -> np.ndarray:
    """Open uniform knot vector on [0,1] with uniform regularity alpha.

    Interior breakpoints are repeated p - alpha times: "the sum of the continuity and the
    multiplicity at a breakpoint is equal to the degree p".
    """
    if p < 0 or not (-1 <= alpha <= p - 1) or n_el < 1:
        raise ValueError("invalid (p, alpha, n_el)")
    interior = np.repeat(np.arange(1, n_el, dtype=np.float64) / n_el, p - alpha)
    return np.concatenate([np.zeros(p + 1), interior, np.ones(p + 1)])


def dimension(p: int, alpha: int, n_el: int) -> int:
    """m = dim S^p_alpha = |Xi| - p - 1."""
    return len(open_uniform_knots(p, alpha, n_el)) - p - 1


def _ratio(num, den):
    """num/den with the paper's convention 0/0 = 0; den == 0 only when num == 0 here."""
    den = np.asarray(den, dtype=np.float64)
    safe = np.where(den == 0.0, 1.0, den)
    return np.where(den == 0.0, 0.0, num / safe)


def basis(xi: np.ndarray, p: int, eta: np.ndarray) -> np.ndarray:
    """All B-splines b_i^p(eta), i = 1..m, by the Cox-de Boor recursion.

    Returns an array of shape (len(eta), m). Degree 0 uses the half-open intervals of
    P:186; at eta = 1 the last non-empty interval is taken closed (left limit), the standard
    convention for open knot vectors.
    """
    eta = np.atleast_1d(np.asarray(eta, dtype=np.float64))
    nk = len(xi)
    # degree 0, functions i = 1..nk-1 (0-based j = 0..nk-2)
    b = np.zeros((len(eta), nk - 1))
    for j in range(nk - 1):
        b[:, j] = (xi[j] <= eta) & (eta < xi[j + 1])
    last = max(j for j in range(nk - 1) if xi[j] < xi[j + 1])
    b[eta == xi[-1], last] = 1.0
    for q in range(1, p + 1):
        nb = np.zeros((len(eta), nk - 1 - q))
        for j in range(nk - 1 - q):
            left = _ratio(eta - xi[j], xi[j + q] - xi[j]) * b[:, j]
            right = _ratio(xi[j + q + 1] - eta, xi[j + q + 1] - xi[j + 1]) * b[:, j + 1]
            nb[:, j] = left + right
        b = nb
    return b


def basis_derivative(xi: np.ndarray, p: int, eta: np.ndarray) -> np.ndarray:
    """First derivatives b_i^p'(eta), shape (len(eta), m).

    Standard derivative of the Cox-de Boor recursion (de Boor, cited at P:180):
    b_i^p' = p/(xi_{i+p}-xi_i) b_i^{p-1} - p/(xi_{i+p+1}-xi_{i+1}) b_{i+1}^{p-1}, 0/0 = 0.
    """
    if p == 0:
        return np.zeros((len(np.atleast_1d(eta)), len(xi) - 1))
    bl = basis(xi, p - 1, eta)  # functions of degree p-1 on the same knots: m+1 of them
    m = len(xi) - p - 1
    d = np.zeros((bl.shape[0], m))
    for j in range(m):
        d[:, j] = (_ratio(p, xi[j + p] - xi[j]) * bl[:, j]
                   - _ratio(p, xi[j + p + 1] - xi[j + 1]) * bl[:, j + 1])
    return d


def gauss_legendre(q: int, a: float = 0.0, b: float = 1.0):
    """q-point Gauss-Legendre rule mapped to [a, b] (numpy's Golub-Welsch-free leggauss)."""
    x, w = np.polynomial.legendre.leggauss(q)
    return 0.5 * (b - a) * x + 0.5 * (a + b), 0.5 * (b - a) * w


def element_quadrature(xi: np.ndarray, q: int):
    """q Gauss points per non-empty knot span (element); nodes strictly inside elements."""
    brk = np.unique(xi)
    xs, ws = [], []
    for a, b in zip(brk[:-1], brk[1:]):
        x, w = gauss_legendre(q, a, b)
        xs.append(x)
        ws.append(w)
    return np.concatenate(xs), np.concatenate(ws)


def greville(xi: np.ndarray, p: int) -> np.ndarray:
    """Greville abscissae g_j = (xi_{j+1} + ... + xi_{j+p}) / p, j = 1..m (for p >= 1).

    Used only for the literal reading of config 3's "nu sampled at dofs".
    """
    m = len(xi) - p - 1
    return np.array([xi[j + 1:j + p + 1].mean() for j in range(m)])
