"""NEXT-3: the Taylor-Hood Stokes system on the eighth of the thick annulus
(§7) and the geometry-aware P_D^G (§6, Appendix),
built from libfdp pieces.

Operator. With r = 1 + eta1, theta = a eta2 (a = pi/4), c = cos theta, s = sin theta, the map
G = (r c, r s, eta3) has J^{-1} = [[c, s, 0], [-s/(a r), c/(a r), 0], [0, 0, 1]], |det J| = a r and
J^{-1} J^{-T} |det J| = diag(a r, 1/(a r), a r). The weak form a(u, v) = int 2 nu grad^s u : grad^s v
 with u = e_s phi_j, v = e_r phi_i gives A_rs = int grad phi_i^T C_rs grad phi_j with
C_rs = |det J| (delta_rs J^{-1} J^{-T} + D_s D_r^T), D_k = J^{-1} e_k (eq. (Q_TH) for r = s),
and B_r = -int rho (D_r . grad phi) |det J|. Every entry is a product r^i cos^j sin^l:
one weighted univariate factor per direction, so each block is a libfdp KronOp whose factors are
libfdp iga_mixed matrices with weights at the iga_quadrature points (q = p + 3 per element,
DESIGN.md N3-4); the whole operator is one grouped kron_ops_apply (krylov._GroupedOperator).

Preconditioner. libfdp iga_geometry_coeffs samples c^k_dd at the quadrature grid,
iga_separable_fit fits tau, mu (log-ALS, N3-2), iga_mixed builds the weighted pencils
K_d = int tau_d b' b', M_d = int mu_d b b, fd_setup solves them; D_V = diag(A_kk) / diag(P^_V,k)
(kron_op_diagonal / fd_operator_diagonal) and D_Q = diag(Q) / diag(P_Q) with Q = int rho rho
|det J| (nu = 1).
"""
from __future__ import annotations

import math

import numpy as np

from . import (FD, FDP_GEOM_ANNULUS, FDP_IGA_INTERIOR, BlockPrecond, KronMass, KronOp,
               iga_geometry_coeffs, iga_mixed, iga_quadrature, iga_separable_fit,
               iga_univariate)
from .krylov import _GroupedOperator

A_ANGLE = math.pi / 4

# a term is (coef, i, j, l): coef * r^i * cos(theta)^j * sin(theta)^l
_DK = {  # (D_k)_d for k, d = 0..2 (lists of terms)
    0: [[(1.0, 0, 1, 0)], [(-1.0 / A_ANGLE, -1, 0, 1)], []],
    1: [[(1.0, 0, 0, 1)], [(1.0 / A_ANGLE, -1, 1, 0)], []],
    2: [[], [], [(1.0, 0, 0, 0)]],
}
_DET = (A_ANGLE, 1, 0, 0)
_GRAM_DET = [(A_ANGLE, 1, 0, 0), (1.0 / A_ANGLE, -1, 0, 0), (A_ANGLE, 1, 0, 0)]  # J^-1 J^-T |det J|


def _mul(*ts):
    c, i, j, l = 1.0, 0, 0, 0
    for t in ts:
        c, i, j, l = c * t[0], i + t[1], j + t[2], l + t[3]
    return (c, i, j, l)


def _coefficient(r: int, s: int):
    """C_rs[d][e] as term lists."""
    C = [[[] for _ in range(3)] for _ in range(3)]
    for d in range(3):
        for e in range(3):
            if r == s and d == e:
                C[d][e].append(_GRAM_DET[d])
            for a in _DK[s][d]:
                for b in _DK[r][e]:
                    C[d][e].append(_mul(_DET, a, b))
    return C


def _weights(term, xq):
    """Per-direction weights of a term at the quadrature points (None = 1)."""
    _, i, j, l = term
    w1 = None if i == 0 else (1.0 + xq) ** i
    w2 = None if (j == 0 and l == 0) else np.cos(A_ANGLE * xq) ** j * np.sin(A_ANGLE * xq) ** l
    return [w1, w2, None]


class AnnulusStokesOperator(_GroupedOperator):
    """y = calA x on the eighth of the thick annulus, TH, nu = 1, x = [u_1 | u_2 | u_3 | p]."""

    def __init__(self, p: int, n_el: int, device: int = 0):
        D = 3
        self.D, self.p, self.n_el = D, p, n_el
        self.q = q = p + 3
        V = (p + 1, p - 1, FDP_IGA_INTERIOR)
        Qs = (p, p - 1, 0)
        xq, _ = iga_quadrature(n_el, q)
        self.xq = xq
        mixed = lambda t, rr, dt, dr, w: iga_mixed(t, rr, n_el, int(dt), int(dr), q, w)
        self.blocks = {}
        for r in range(D):
            for s in range(D):
                C = _coefficient(r, s)
                terms, coef = [], []
                for d in range(D):
                    for e in range(D):
                        for t in C[d][e]:
                            w = _weights(t, xq)
                            terms.append([mixed(V, V, m == d, m == e, w[m]) for m in range(D)])
                            coef.append(t[0])
                self.blocks[(r, s)] = KronOp(terms, coef, device)
        self.B, self.BT = [], []
        for r in range(D):
            terms, coef = [], []
            for d in range(D):
                for a in _DK[r][d]:
                    t = _mul(_DET, a)
                    w = _weights(t, xq)
                    terms.append([mixed(Qs, V, False, m == d, w[m]) for m in range(D)])
                    coef.append(-t[0])
            self.B.append(KronOp(terms, coef, device))
            self.BT.append(KronOp([[np.asfortranarray(f.T) for f in F] for F in terms], coef, device))
        w = _weights(_DET, xq)
        self.Q = KronOp([[mixed(Qs, Qs, False, False, w[m]) for m in range(D)]], [_DET[0]], device)
        self.vel_dims = [self.blocks[(k, k)].nin for k in range(D)]
        self.q_dims = self.B[0].nout
        group = []
        for r in range(D):
            for s in range(D):
                group.append((self.blocks[(r, s)], s, r))
            group.append((self.BT[r], D, r))
        for r in range(D):
            group.append((self.B[r], r, D))
        sizes = [int(np.prod(v)) for v in self.vel_dims] + [int(np.prod(self.q_dims))]
        self._finalize(group, sizes, device)
        self.device = device


def geometry_block(op: AnnulusStokesOperator, max_sweeps: int = 50, tol: float = 1e-8):
    """The geometry-aware P_D^G for ``op`` (Appendix + §6): returns (BlockPrecond, info)."""
    D, p, n_el, q = op.D, op.p, op.n_el, op.q
    V = (p + 1, p - 1, FDP_IGA_INTERIOR)
    x = op.xq
    nq = x.size
    fds, dv, sweeps = [], [], []
    for k in range(D):
        c = iga_geometry_coeffs(FDP_GEOM_ANNULUS, D, k, x)
        tau, mu, sw = iga_separable_fit(c, [nq] * D, max_sweeps, tol)
        sweeps.append(sw)
        Ks = [iga_mixed(V, V, n_el, 1, 1, q, tau[d]) for d in range(D)]
        Ms = [iga_mixed(V, V, n_el, 0, 0, q, mu[d]) for d in range(D)]
        f = FD(Ks, Ms, [1.0] * D, device=op.device)
        fds.append(f)
        dv.append(op.blocks[(k, k)].diagonal() / f.operator_diagonal())
    _, Mq = iga_univariate(p, p - 1, n_el)
    PQ = KronOp([[Mq] * D], [1.0], op.device)
    dq = op.Q.diagonal() / PQ.diagonal()
    blk = BlockPrecond(fds, KronMass([Mq] * D, device=op.device), np.concatenate(dv), dq)
    return blk, {"fit_sweeps": sweeps}


def plain_block(op: AnnulusStokesOperator):
    """The geometry-free P_D: the parametric-domain TH pencils."""
    from . import build_block, discretization
    return build_block(discretization(op.D, "TH", op.p, op.n_el), device=op.device)
