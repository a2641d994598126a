"""Matrix-free Stokes system on the unit cube / square (identity map, nu = 1) in Kronecker form,
for the MINRES iteration-count harness. Oracle only (test infrastructure).

From PAPER.md §3: a(w, v) = int 2 grad^s w : grad^s v, b(v, q) = -int q div v,
system [[A, B^T], [B, 0]]. With w = e_s phi_j, v = e_r phi_i,
2 grad^s(e_s phi_j) : grad^s(e_r phi_i) = delta_rs grad phi_i . grad phi_j + d_s phi_i d_r phi_j,
so A_kk = P_V,k and, for r != s, A_rs[i, j] = int d_s phi_i d_r phi_j -- a single
Kronecker product with G^(test,trial) = int b'_test b_trial in direction s, its mirror in
direction r and a mass factor elsewhere. B_r[l, j] = -int rho_l d_r phi_j. On the cube the RT
Nitsche form sigma has no cross-component terms (the tangential derivatives of a
normal component vanish on the faces where it is restricted), so A_rs^RT has the same form.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import splines, univariate


def _space(deg, alpha, n_el, interior):
    xi = splines.open_uniform_knots(deg, alpha, n_el)
    return xi, deg, interior


def _mixed(test, trial, n_el, q, dtest=False, dtrial=False, weight=None):
    """M[l, m] = int wt(x) (b^test_l)^(') (b^trial_m)^(') over [0,1] by element Gauss quadrature
    (wt = 1 unless a weight function is given)."""
    xt, dt, it = test
    xr, dr, ir = trial
    x, w = splines.element_quadrature(np.linspace(0, 1, n_el + 1), q)
    if weight is not None:
        w = w * weight(x)
    Bt = splines.basis_derivative(xt, dt, x) if dtest else splines.basis(xt, dt, x)
    Br = splines.basis_derivative(xr, dr, x) if dtrial else splines.basis(xr, dr, x)
    if it:
        Bt = Bt[:, 1:-1]
    if ir:
        Br = Br[:, 1:-1]
    return Bt.T @ (w[:, None] * Br)


def _kron_apply(factors, x):
    """(F_D (x) .. (x) F_1) x for rectangular factors F_d (n_out_d x n_in_d), F[0] acts on i1."""
    dims_in = [F.shape[1] for F in factors]
    X = np.reshape(x, dims_in, order="F")
    for d, F in enumerate(factors):
        Xd = np.moveaxis(X, d, 0)
        sh = Xd.shape
        Y = F @ Xd.reshape(sh[0], -1)
        X = np.moveaxis(Y.reshape((F.shape[0],) + sh[1:]), 0, d)
    return np.reshape(X, -1, order="F")


class StokesCube:
    """y = calA x for x = [u_1 | .. | u_D | p] (vec order, i1 fastest).

    nu_terms: separable viscosity nu(x) = sum_t c_t prod_d w_{t,d}(x_d) as [(c_t, [w_t1, ..]), ..]
    (None = constant 1). Config 3's nu = 1 + 0.5 sin(2 pi x) sin(2 pi y) sin(2 pi z) is two
    terms; it equals 1 on the boundary of the cube, so the Nitsche terms keep weight 1."""

    def __init__(self, D: int, disc: str, p: int, n_el: int, nu_terms=None, rt_own_alpha=None):
        """rt_own_alpha: regularity of the RT own direction (default alpha + 1; p - 1 is
        config 3's literal "C^3" wording)."""
        self.D = D
        alpha = p - 1
        nu_terms = nu_terms or [(1.0, None)]
        weighted = any(ws is not None for _, ws in nu_terms)
        # exact for products of degree <= p+1 splines and derivatives (C-4); extra points for
        # non-polynomial weights
        q = p + 3 + (4 if weighted else 0)
        Q = _space(p, alpha, n_el, False)
        if disc == "TH":
            V = [[_space(p + 1, alpha, n_el, True)] * D for _ in range(D)]
        elif disc == "RT":
            N = _space(p + 1, alpha + 1 if rt_own_alpha is None else rt_own_alpha, n_el, True)
            T = _space(p, alpha, n_el, False)
            V = [[N if d == k else T for d in range(D)] for k in range(D)]
        else:
            raise ValueError(disc)
        cp = univariate.c_pen(p)
        self.vel_dims = [[_mixed(V[k][d], V[k][d], n_el, q).shape[0] for d in range(D)] for k in range(D)]
        self.q_dims = [_mixed(Q, Q, n_el, q).shape[0]] * D
        # diagonal blocks: A_kk = sum_t c_t sum_d c_d (x) (K_w at d, M_w elsewhere); the RT
        # tangential K~ carries the Nitsche bracket in the constant (boundary weight 1) term only
        self.diag = []   # per k: list of (scalar, factors) Kronecker terms
        for k in range(D):
            terms = []
            for ct, ws in nu_terms:
                wt = (lambda d: None) if ws is None else (lambda d, ws=ws: ws[d])
                Ms = [sp.csr_matrix(_mixed(V[k][d], V[k][d], n_el, q, weight=wt(d))) for d in range(D)]
                Ks = []
                for d in range(D):
                    if disc == "RT" and d != k and ws is None:
                        Ks.append(sp.csr_matrix(univariate.nitsche_stiffness(p, alpha, n_el, cp)))
                    else:
                        Ks.append(sp.csr_matrix(_mixed(V[k][d], V[k][d], n_el, q, True, True, weight=wt(d))))
                for d in range(D):
                    terms.append((ct * (1.0 + (d == k)), [Ks[e] if e == d else Ms[e] for e in range(D)]))
            self.diag.append(terms)
        # off-diagonal A_rs (test component r, trial component s), r != s: int nu d_s phi_i d_r phi_j
        self.off = {}
        for r in range(D):
            for s in range(D):
                if r == s:
                    continue
                terms = []
                for ct, ws in nu_terms:
                    F = []
                    for d in range(D):
                        wd = None if ws is None else ws[d]
                        F.append(sp.csr_matrix(_mixed(V[r][d], V[s][d], n_el, q, dtest=(d == s),
                                                      dtrial=(d == r), weight=wd)))
                    terms.append((ct, F))
                self.off[(r, s)] = terms
        # divergence blocks B_r = -( (x) D^QV at r, M^QV elsewhere )
        self.B = []
        for r in range(D):
            F = [_mixed(Q, V[r][d], n_el, q, dtrial=(d == r)) for d in range(D)]
            self.B.append([sp.csr_matrix(f) for f in F])
        self.sizes = [int(np.prod(v)) for v in self.vel_dims] + [int(np.prod(self.q_dims))]
        self.off_idx = np.concatenate([[0], np.cumsum(self.sizes)]).astype(np.int64)
        self.n = int(self.off_idx[-1])

    def _blk(self, x, k):
        return x[self.off_idx[k]:self.off_idx[k + 1]]

    def B_apply(self, u):
        """B u = sum_r B_r u_r (velocity [u_1 | .. | u_D] -> pressure), B_r = -(x) D^QV / M^QV."""
        yp = np.zeros(self.sizes[self.D])
        for r in range(self.D):
            yp -= _kron_apply(self.B[r], self._blk(u, r))
        return yp

    def BT_apply(self, pr):
        """B^T p = [B_1^T p | .. | B_D^T p] (pressure -> velocity)."""
        return np.concatenate([-_kron_apply([f.T.tocsr() for f in self.B[r]], pr) for r in range(self.D)])

    def matvec(self, x):
        D = self.D
        y = np.zeros_like(x)
        u = [self._blk(x, k) for k in range(D)]
        pr = self._blk(x, D)
        for r in range(D):
            acc = np.zeros(self.sizes[r])
            for c, F in self.diag[r]:
                acc += c * _kron_apply(F, u[r])
            for s in range(D):
                if s != r:
                    for c, F in self.off[(r, s)]:
                        acc += c * _kron_apply(F, u[s])
            # B_r^T p
            acc -= _kron_apply([f.T.tocsr() for f in self.B[r]], pr)
            y[self.off_idx[r]:self.off_idx[r + 1]] = acc
        yp = np.zeros(self.sizes[D])
        for r in range(D):
            yp -= _kron_apply(self.B[r], u[r])
        y[self.off_idx[D]:] = yp
        return y


def project_rhs(f: np.ndarray, n_pressure: int) -> np.ndarray:
    """Make f consistent with the singular system: remove the component along the pressure null
    vector (0, 1) (no zero-mean constraint is imposed on the space)."""
    g = np.array(f, dtype=np.float64, copy=True)
    g[-n_pressure:] -= g[-n_pressure:].mean()
    return g


def config3_nu_terms(D: int = 3):
    """nu(x) = 1 + 0.5 prod_d sin(2 pi x_d) (synth.viscosity) as two separable terms."""
    s = lambda x: np.sin(2 * np.pi * x)
    return [(1.0, None), (0.5, [s] * D)]


def _kron_diag(diags):
    """diag(F_D (x) .. (x) F_1) from per-direction diagonals [d_1, .., d_D], vec order (i1 fastest)."""
    out = np.ones(1)
    for dg in diags:
        out = np.kron(dg, out)
    return out


def nu_scalings_paper(disc, op: StokesCube, nu, q: int):
    """Config 3 under the paper's definition of the P^G scalings (second row;
    PAPER.md §6): [D_V]_ii = [A_kk]_ii / [P_V,k]_ii with A_kk the nu-weighted
    velocity block of ``op`` (built with the separable nu terms), and [D_Q]_ii = [Q]_ii / [P_Q]_ii
    with Q = int nu^{-1} rho_i rho_j (identity map). diag(A_kk) is the Kronecker product
    of the factors' diagonals summed over the terms; diag(Q) is the q-point element Gauss rule in
    every direction applied to nu^{-1} rho_i^2 on the tensor grid (nu^{-1} is not separable), as
    three tensor contractions; nu is the callable nu(x, y, z) (C-6b)."""
    D = disc.D
    dv = []
    for k, c in enumerate(disc.comps):
        dA = np.zeros(c.size)
        for cf, F in op.diag[k]:
            dA += cf * _kron_diag([np.asarray(f.diagonal()).ravel() for f in F])
        dP = np.zeros(c.size)
        for d in range(D):
            dP += c.coef[d] * _kron_diag([np.diag(c.Ks[e]) if e == d else np.diag(c.Ms[e]) for e in range(D)])
        dv.append(dA / dP)
    xi = splines.open_uniform_knots(disc.p, disc.p - 1, disc.n_el)
    x, w = splines.element_quadrature(np.linspace(0, 1, disc.n_el + 1), q)
    E = w[:, None] * splines.basis(xi, disc.p, x) ** 2        # (points, n_q): w_g b_i(x_g)^2
    G = np.meshgrid(*([x] * D), indexing="ij")
    T = 1.0 / nu(*G)                                            # nu^{-1} on the grid, [g1, .., gD]
    for d in range(D):                                          # contract g_d against E
        T = np.moveaxis(np.tensordot(E, T, axes=([0], [d])), 0, d)
    dQ = np.reshape(T, -1, order="F")
    dPq = _kron_diag([np.diag(M) for M in disc.Mq])
    return np.concatenate(dv), dQ / dPq
