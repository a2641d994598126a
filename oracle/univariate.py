"""Univariate stiffness/mass factors (§5). Oracle only."""
from __future__ import annotations

import numpy as np

from . import splines


def c_pen(p: int) -> float:
    """Nitsche penalty C_pen = 5(alpha + 1) with alpha = p - 1, p the pressure degree."""
    return 5.0 * p


def stiffness_mass(deg: int, alpha: int, n_el: int, q: int | None = None):
    """Full-space K[l,s] = int b_l' b_s', M[l,s] = int b_l b_s over [0,1].

    Element-wise Gauss quadrature with q = deg + 1 points: exact for the
    polynomial integrands of degree 2*deg and 2*deg - 2.
    """
    xi = splines.open_uniform_knots(deg, alpha, n_el)
    q = deg + 1 if q is None else q
    x, w = splines.element_quadrature(xi, q)
    B = splines.basis(xi, deg, x)
    dB = splines.basis_derivative(xi, deg, x)
    M = B.T @ (w[:, None] * B)
    K = dB.T @ (w[:, None] * dB)
    return K, M


def interior(A: np.ndarray) -> np.ndarray:
    """Restriction to l, s = 2..m-1 (Dirichlet / normal-trace basis)."""
    return A[1:-1, 1:-1]


def nitsche_stiffness(deg: int, alpha: int, n_el: int, cpen: float, q: int | None = None):
    """K-tilde of P:701-704 on the full tangential space S^deg_alpha (l, s = 1..m).

    K~[l,s] = int b_l' b_s' - [ b_l'(1) b_s(1) - b_l'(0) b_s(0) + b_s'(1) b_l(1)
                                - b_s'(0) b_l(0) - 2 (C_pen/h) (b_l(1) b_s(1) + b_l(0) b_s(0)) ],
    with h = 1/n_el (uniform mesh size).
    """
    K, _ = stiffness_mass(deg, alpha, n_el, q)
    xi = splines.open_uniform_knots(deg, alpha, n_el)
    ends = np.array([0.0, 1.0])
    b = splines.basis(xi, deg, ends)             # rows: eta=0, eta=1
    db = splines.basis_derivative(xi, deg, ends)
    b0, b1, d0, d1 = b[0], b[1], db[0], db[1]
    h = 1.0 / n_el
    bracket = (np.outer(d1, b1) - np.outer(d0, b0) + np.outer(b1, d1) - np.outer(b0, d0)
               - 2.0 * (cpen / h) * (np.outer(b1, b1) + np.outer(b0, b0)))
    return K - bracket


def th_velocity_pencil(p: int, n_el: int):
    """(K_k^TH, M_k^TH): degree p+1, regularity alpha = p-1, interior l,s = 2..m-1."""
    K, M = stiffness_mass(p + 1, p - 1, n_el)
    return interior(K), interior(M)


def rt_normal_pencil(p: int, n_el: int, alpha_own: int | None = None):
    """(K_k^RT, M_k^RT): degree p+1, regularity alpha+1 = p, interior. alpha_own
    overrides the regularity (SURVEY.md C-3's literal reading of config 3: p - 1)."""
    K, M = stiffness_mass(p + 1, p if alpha_own is None else alpha_own, n_el)
    return interior(K), interior(M)


def rt_tangential_pencil(p: int, n_el: int):
    """(K~_k^RT, M~_k^RT): degree p, regularity alpha = p-1, full space, Nitsche."""
    Kt = nitsche_stiffness(p, p - 1, n_el, c_pen(p))
    _, Mt = stiffness_mass(p, p - 1, n_el)
    return Kt, Mt


def pressure_mass(p: int, n_el: int) -> np.ndarray:
    """M_k of P_Q = M_3 (x) M_2 (x) M_1: degree p, regularity alpha, full."""
    return stiffness_mass(p, p - 1, n_el)[1]
