"""Mapped geometry and geometry-aware pencils. Oracle only (test
infrastructure; imported by tests/ only).

PAPER.md passages followed:
  * eq. (Q_TH): A_kk^TH = int grad B_i^T C_k grad B_j with
    C_k = nu (J^{-1} J^{-T} + D_k D_k^T) |det J|, D_k = J^{-1} e_k; the off-diagonal blocks follow
    from the same weak form a(u, v) = int 2 nu grad^s u : grad^s v with u = e_s phi_j,
    v = e_r phi_i: C_rs = nu |det J| (delta_rs J^{-1} J^{-T} + D_s D_r^T) (N3-1);
    B_r = -int rho (D_r . grad phi) |det J| (b(v, q) = -int q div v).
  * §6: P_Q^G = D_Q^{1/2} P_Q D_Q^{1/2}, [D_Q]_ii = [Q]_ii / [P_Q]_ii;
    P_V^G = D_V^{1/2} P^_V D_V^{1/2}, [D_V]_ii = [A]_ii / [P^_V]_ii.
  * Appendix: drop the off-diagonal entries of C_k, approximate
    c^k_dd ~ tau_d(eta_d) prod_{m != d} mu_m(eta_m) at the quadrature points, and build the
    weighted pencils K^k_d = int tau_d b' b', M^k_d = int mu_d b b (TH).
  * §7: the eighth of a thick annulus, inner radius 1, outer radius 2, height 1.

Readings: the annulus map G(eta) = ((1+eta1) cos(pi eta2 / 4),
(1+eta1) sin(pi eta2 / 4), eta3) (N3-3); the separable fit is log-domain alternating least
squares (N3-2; the paper cites sup-norm separation algorithms without operational detail);
TH only (RT on mapped domains needs the Hessian terms of eq. (Akk_RT), out of scope).

Every metric quantity of the annulus is a product of univariate functions, so C_rs, B_r and Q
are sums of Kronecker products of weighted univariate matrices: ``Sep`` holds such separable
expansions symbolically (no trigonometric simplification) so that the Kronecker operator is
derived mechanically from J^{-1} and det J; tests pin it against brute-force 3D quadrature of
the weak form with a numerically inverted Jacobian.
"""
from __future__ import annotations

import math

import numpy as np

from . import splines, univariate
from .stokes import _kron_apply, _mixed, _space


class Sep:
    """sum_t c_t prod_m f_tm(eta_m) (f = None means 1); D = number of directions."""

    def __init__(self, D, terms=None):
        self.D = D
        self.terms = list(terms or [])

    @staticmethod
    def const(D, c):
        return Sep(D, [(float(c), (None,) * D)] if c != 0 else [])

    @staticmethod
    def univ(D, m, f):
        fs = [None] * D
        fs[m] = f
        return Sep(D, [(1.0, tuple(fs))])

    def __add__(self, o):
        return Sep(self.D, self.terms + o.terms)

    def __neg__(self):
        return Sep(self.D, [(-c, f) for c, f in self.terms])

    def __sub__(self, o):
        return self + (-o)

    def scale(self, s):
        return Sep(self.D, [(s * c, f) for c, f in self.terms])

    def __mul__(self, o):
        out = []
        for c1, f1 in self.terms:
            for c2, f2 in o.terms:
                fs = []
                for a, b in zip(f1, f2):
                    if a is None:
                        fs.append(b)
                    elif b is None:
                        fs.append(a)
                    else:
                        fs.append(lambda x, a=a, b=b: a(x) * b(x))
                out.append((c1 * c2, tuple(fs)))
        return Sep(self.D, out)

    def __call__(self, *eta):
        v = 0.0
        for c, fs in self.terms:
            t = c
            for f, x in zip(fs, eta):
                if f is not None:
                    t = t * f(x)
            v = v + t
        return v


class Geometry:
    """A map G of [0,1]^D with J^{-1} (J[a, b] = dG_a / d eta_b) and |det J| as Sep expansions and
    G itself as a plain function (for the brute-force pins)."""

    def __init__(self, D, G, Jinv, detJ, name):
        self.D, self.G, self.Jinv, self.detJ, self.name = D, G, Jinv, detJ, name


def identity(D: int = 3) -> Geometry:
    Jinv = [[Sep.const(D, 1.0 if a == b else 0.0) for b in range(D)] for a in range(D)]
    return Geometry(D, lambda *e: np.stack(e), Jinv, Sep.const(D, 1.0), "identity")


ANNULUS_ANGLE = math.pi / 4  # an eighth of the full annulus


def annulus() -> Geometry:
    """Eighth of the thick annulus: r = 1 + eta1 in [1, 2], theta = (pi/4) eta2,
    z = eta3. J = [[cos, -a r sin, 0], [sin, a r cos, 0], [0, 0, 1]] (a = pi/4), so
    J^{-1} = [[cos, sin, 0], [-sin/(a r), cos/(a r), 0], [0, 0, 1]] and det J = a r."""
    D = 3
    a = ANNULUS_ANGLE
    c = Sep.univ(D, 1, lambda y: np.cos(a * y))
    s = Sep.univ(D, 1, lambda y: np.sin(a * y))
    rinv = Sep.univ(D, 0, lambda x: 1.0 / (1.0 + x))
    r = Sep.univ(D, 0, lambda x: 1.0 + x)
    z = Sep.const(D, 0.0)
    one = Sep.const(D, 1.0)
    Jinv = [[c, s, z],
            [(s * rinv).scale(-1.0 / a), (c * rinv).scale(1.0 / a), z],
            [z, z, one]]

    def G(e1, e2, e3):
        rr = 1.0 + e1
        return np.stack([rr * np.cos(a * e2), rr * np.sin(a * e2), e3 + 0.0 * e1])

    return Geometry(D, G, Jinv, r.scale(a), "annulus")


def coefficient(geo: Geometry, r: int, s: int, nu: Sep | None = None):
    """C_rs[d][e] (Sep) with A_rs[i, j] = int sum_de C_rs[d][e] d_d phi_i d_e phi_j (test
    component r, trial component s): nu |det J| (delta_rs J^{-1} J^{-T} + D_s D_r^T),
    D_k = J^{-1} e_k (eq. (Q_TH) for r = s = k)."""
    D = geo.D
    Ji = geo.Jinv
    C = [[Sep(D) for _ in range(D)] for _ in range(D)]
    for d in range(D):
        for e in range(D):
            t = Sep(D)
            if r == s:
                for m in range(D):
                    t = t + Ji[d][m] * Ji[e][m]
            t = t + Ji[d][s] * Ji[e][r]
            t = t * geo.detJ
            if nu is not None:
                t = t * nu
            C[d][e] = t
    return C


class StokesMapped:
    """Taylor-Hood Stokes system [[A, B^T], [B, 0]] on a mapped domain with a separable metric, as
    sums of Kronecker products of weighted univariate matrices (quadrature: q = p + 3 Gauss points
    per element, the grid where the weights are sampled; N3-4)."""

    def __init__(self, geo: Geometry, p: int, n_el: int, q: int | None = None):
        D = geo.D
        self.D, self.geo, self.p, self.n_el = D, geo, p, n_el
        self.q = q or p + 3
        alpha = p - 1
        self.Vsp = _space(p + 1, alpha, n_el, True)
        self.Qsp = _space(p, alpha, n_el, False)
        mixed = lambda t, rr, dt, dr, w: _mixed(t, rr, n_el, self.q, dtest=dt, dtrial=dr, weight=w)
        self.blocks = {}
        for r in range(D):
            for s in range(D):
                C = coefficient(geo, r, s)
                terms = []
                for d in range(D):
                    for e in range(D):
                        for cf, fs in C[d][e].terms:
                            F = [mixed(self.Vsp, self.Vsp, m == d, m == e, fs[m]) for m in range(D)]
                            terms.append((cf, F))
                self.blocks[(r, s)] = terms
        self.B = []
        for r in range(D):
            terms = []
            for d in range(D):
                t = geo.Jinv[d][r] * geo.detJ            # (D_r)_d |det J|
                for cf, fs in t.terms:
                    F = [mixed(self.Qsp, self.Vsp, False, m == d, fs[m]) for m in range(D)]
                    terms.append((-cf, F))
            self.B.append(terms)
        nv = _mixed(self.Vsp, self.Vsp, n_el, self.q).shape[0]
        nq = _mixed(self.Qsp, self.Qsp, n_el, self.q).shape[0]
        self.vel_dims = [[nv] * D for _ in range(D)]
        self.q_dims = [nq] * D
        self.sizes = [nv ** D] * D + [nq ** D]
        self.off_idx = np.concatenate([[0], np.cumsum(self.sizes)]).astype(np.int64)
        self.n = int(self.off_idx[-1])

    def _blk(self, x, k):
        return x[self.off_idx[k]:self.off_idx[k + 1]]

    def matvec(self, x):
        D = self.D
        y = np.zeros_like(x)
        pr = self._blk(x, D)
        for r in range(D):
            acc = np.zeros(self.sizes[r])
            for s in range(D):
                for c, F in self.blocks[(r, s)]:
                    acc += c * _kron_apply(F, self._blk(x, s))
            for c, F in self.B[r]:
                acc += c * _kron_apply([f.T for f in F], pr)
            y[self.off_idx[r]:self.off_idx[r + 1]] = acc
        yp = np.zeros(self.sizes[D])
        for r in range(D):
            for c, F in self.B[r]:
                yp += c * _kron_apply(F, self._blk(x, r))
        y[self.off_idx[D]:] = yp
        return y

    def B_apply(self, u):
        """B u = sum_r B_r u_r (velocity -> pressure)."""
        yp = np.zeros(self.sizes[self.D])
        for r in range(self.D):
            for c, F in self.B[r]:
                yp += c * _kron_apply(F, self._blk(u, r))
        return yp

    def BT_apply(self, pr):
        """B^T p = [B_1^T p | .. | B_D^T p]."""
        out = []
        for r in range(self.D):
            acc = np.zeros(self.sizes[r])
            for c, F in self.B[r]:
                acc += c * _kron_apply([f.T for f in F], pr)
            out.append(acc)
        return np.concatenate(out)

    def diag_A(self, k):
        """diag(A_kk) = sum_terms c prod_m diag(F_m) (Kronecker product of diagonals, i1 fastest)."""
        out = np.zeros(self.sizes[k])
        for c, F in self.blocks[(k, k)]:
            dg = np.ones(1)
            for f in F:
                dg = np.kron(np.diag(f), dg)
            out += c * dg
        return out

    def diag_Q(self):
        """diag(Q), Q = int nu^{-1} rho_i rho_j dx = int rho_i rho_j |det J| (nu = 1)."""
        out = np.zeros(self.sizes[-1])
        for c, fs in self.geo.detJ.terms:
            dg = np.ones(1)
            for m in range(self.D):
                dg = np.kron(np.diag(_mixed(self.Qsp, self.Qsp, self.n_el, self.q, weight=fs[m])), dg)
            out += c * dg
        return out


def quadrature_grid(n_el: int, q: int):
    """1D element Gauss points / weights on the uniform mesh (the sampling grid)."""
    return splines.element_quadrature(np.linspace(0, 1, n_el + 1), q)


def sample_diagonal(geo: Geometry, k: int, x: np.ndarray):
    """c^k_dd at the tensor grid x (same 1D points per direction), arrays indexed [i1, i2, i3]."""
    C = coefficient(geo, k, k)
    E = np.meshgrid(*([x] * geo.D), indexing="ij")
    return [np.broadcast_to(np.asarray(C[d][d](*E), dtype=np.float64), E[0].shape).copy()
            for d in range(geo.D)]


def separable_fit(c, max_sweeps: int = 50, tol: float = 1e-8):
    """Log-domain alternating least squares (N3-2): minimise
    sum_d || log c_d - (log tau_d(i_d) + sum_{m != d} log mu_m(i_m)) ||^2 over the grid.
    Init mu = 1, log tau_d(i) = mean over the slice i_d = i of log c_d. Each sweep updates
    tau_1..tau_D, then mu_1..mu_D, each by its closed-form slice mean with the others fixed. Gauge:
    every mu has geometric mean 1 (the scale moves into the tau's). Stops when the objective's
    relative change is <= tol or after max_sweeps. Returns (tau, mu, objective history)."""
    D = len(c)
    L = [np.log(ci) for ci in c]
    shape = L[0].shape
    lt = []
    for d in range(D):
        ax = tuple(a for a in range(D) if a != d)
        lt.append(L[d].mean(axis=ax))
    lm = [np.zeros(shape[m]) for m in range(D)]

    def expand(v, m):
        sh = [1] * D
        sh[m] = shape[m]
        return v.reshape(sh)

    def model(d, skip=None):
        t = expand(lt[d], d)
        for m in range(D):
            if m != d and m != skip:
                t = t + expand(lm[m], m)
        return t

    def objective():
        return float(sum(((L[d] - model(d)) ** 2).sum() for d in range(D)))

    hist = [objective()]
    for _ in range(max_sweeps):
        for d in range(D):
            ax = tuple(a for a in range(D) if a != d)
            lt[d] = (L[d] - (model(d) - expand(lt[d], d))).mean(axis=ax)
        for m in range(D):
            ax = tuple(a for a in range(D) if a != m)
            acc = np.zeros(shape[m])
            cnt = 0
            for d in range(D):
                if d == m:
                    continue
                acc = acc + (L[d] - model(d, skip=m)).mean(axis=ax)
                cnt += 1
            lm[m] = acc / cnt
        for m in range(D):  # gauge: geometric mean of mu_m = 1
            g = lm[m].mean()
            lm[m] = lm[m] - g
            for d in range(D):
                if d != m:
                    lt[d] = lt[d] + g
        hist.append(objective())
        if abs(hist[-2] - hist[-1]) <= tol * max(abs(hist[-2]), 1e-300):
            break
    return [np.exp(v) for v in lt], [np.exp(v) for v in lm], hist


def geo_pencils(tau, mu, p: int, n_el: int, q: int):
    """Weighted TH pencils of the Appendix: K_d = int tau_d b' b', M_d = int mu_d b b
    on degree p+1, regularity p-1, interior functions; tau, mu are node values at the element
    Gauss points (q per element), the grid they were fitted on."""
    xi = splines.open_uniform_knots(p + 1, p - 1, n_el)
    x, w = quadrature_grid(n_el, q)
    B = splines.basis(xi, p + 1, x)[:, 1:-1]
    dB = splines.basis_derivative(xi, p + 1, x)[:, 1:-1]
    Ks = [dB.T @ ((w * t)[:, None] * dB) for t in tau]
    Ms = [B.T @ ((w * m)[:, None] * B) for m in mu]
    return Ks, Ms


def geo_discretization(op: StokesMapped):
    """The geometry-aware P_D^G of §6 + Appendix for the TH system ``op``: per component k the
    separable fit of c^k_dd, the weighted pencils (coefficients 1: the factor 2 of the identity
    case now lives in tau), D_V = diag(A_kk) / diag(P^_V,k), and D_Q = diag(Q) / diag(P_Q).
    Returns (spaces.Discretization, D_V, D_Q)."""
    from . import spaces
    D, p, n_el, q = op.D, op.p, op.n_el, op.q
    x, _ = quadrature_grid(n_el, q)
    comps, dv = [], []
    for k in range(D):
        tau, mu, _ = separable_fit(sample_diagonal(op.geo, k, x))
        Ks, Ms = geo_pencils(tau, mu, p, n_el, q)
        coef = [1.0] * D
        dP = np.zeros(op.sizes[k])
        for d in range(D):
            dg = np.ones(1)
            for m in range(D):
                dg = np.kron(np.diag(Ks[m] if m == d else Ms[m]), dg)
            dP += dg
        dv.append(op.diag_A(k) / dP)
        comps.append(spaces.Component(Ks, Ms, coef, [None] * D))
    Mq = univariate.pressure_mass(p, n_el)
    dPq = np.ones(1)
    for _ in range(D):
        dPq = np.kron(np.diag(Mq), dPq)
    dq = op.diag_Q() / dPq
    disc = spaces.Discretization(D, "TH", p, n_el, comps, [Mq] * D, [None] * D)
    return disc, np.concatenate(dv), dq


def plain_discretization(op: StokesMapped):
    """The geometry-free P_D (parametric-domain pencils, P:1063-1069 without the G): the cube's
    TH pencils for the same degree and mesh."""
    from . import spaces
    return spaces.build(op.D, "TH", op.p, op.n_el)
