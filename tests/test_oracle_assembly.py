"""Brute-force 3D quadrature pins for coefficient placement and Kronecker factor ordering.

The blocks P_V,k are *defined* as bilinear forms: TH
[P_V,k]_ij = a^(e_k B_i, e_k B_j) with a^(w,v) = int 2 grad^s w : grad^s v; RT adds sigma^(w,v)
(P:658-659). Here those integrals are evaluated directly at 3D / face quadrature points from
trivariate basis values (products of univariate B-splines), without any Kronecker
structure, and compared with the oracle's Kronecker sums -- a wrong coefficient,
a transposed factor order or a wrong K~ sign fails.
"""
import itertools

import numpy as np
import pytest

from oracle import fd, kron, splines, univariate


def _space(deg, alpha, n_el, interior):
    xi = splines.open_uniform_knots(deg, alpha, n_el)
    sl = slice(1, -1) if interior else slice(None)
    return xi, deg, sl


def _eval(space, x):
    xi, deg, sl = space
    return splines.basis(xi, deg, x)[:, sl], splines.basis_derivative(xi, deg, x)[:, sl]


def _trivariate(spaces3, pts):
    """B_i(eta) and grad B_i(eta) at 3D points for all dofs i in vec order (i1 fastest)."""
    vals = [_eval(spaces3[d], pts[:, d]) for d in range(3)]
    n = [v[0].shape[1] for v in vals]
    N = n[0] * n[1] * n[2]
    B = np.zeros((len(pts), N))
    G = np.zeros((len(pts), N, 3))
    for i3, i2, i1 in itertools.product(range(n[2]), range(n[1]), range(n[0])):
        i = i1 + n[0] * (i2 + n[1] * i3)
        b = [vals[0][0][:, i1], vals[1][0][:, i2], vals[2][0][:, i3]]
        db = [vals[0][1][:, i1], vals[1][1][:, i2], vals[2][1][:, i3]]
        B[:, i] = b[0] * b[1] * b[2]
        G[:, i, 0] = db[0] * b[1] * b[2]
        G[:, i, 1] = b[0] * db[1] * b[2]
        G[:, i, 2] = b[0] * b[1] * db[2]
    return B, G, n


def _grid(n_els, q):
    xs, ws = [], []
    for n_el in n_els:
        x, w = splines.element_quadrature(np.linspace(0, 1, n_el + 1), q)
        xs.append(x)
        ws.append(w)
    X = np.array(list(itertools.product(*xs)))
    W = np.array([a * b * c for a, b, c in itertools.product(*ws)])
    return X, W


def _a_hat(G, W, k):
    """int 2 grad^s(e_k B_i) : grad^s(e_k B_j) straight from the definition of a^."""
    N = G.shape[1]
    A = np.zeros((N, N))
    ek = np.eye(3)[k]
    for q in range(len(W)):
        S = []
        for i in range(N):
            gw = np.outer(ek, G[q, i])           # grad w, w = e_k B_i: (grad w)_{ab} = d_b w_a
            S.append(0.5 * (gw + gw.T))
        S = np.array(S)                          # (N, 3, 3)
        A += W[q] * 2.0 * np.einsum("iab,jab->ij", S, S)
    return A


@pytest.mark.parametrize("k", [0, 1, 2])
def test_th_block_equals_kronecker_sum(k):
    p = 1   # velocity degree 2, regularity 0 (alpha = p - 1)
    n_els = (2, 3, 1)  # anisotropic on purpose: dims (3, 5, 1)
    sp = [_space(p + 1, p - 1, n, True) for n in n_els]
    X, W = _grid(n_els, p + 3)
    _, G, n = _trivariate(sp, X)
    A = _a_hat(G, W, k)
    Ks, Ms = zip(*[univariate.th_velocity_pencil(p, ne) for ne in n_els])
    coef = [1.0 + (d == k) for d in range(3)]
    R = fd.assemble_R(list(Ks), list(Ms), coef)
    assert np.max(np.abs(A - R)) < 1e-13 * np.max(np.abs(R))


@pytest.mark.parametrize("k,own", [(0, None), (1, None), (2, None), (0, 1), (2, 1)])
def test_rt_block_equals_kronecker_sum_with_nitsche(k, own):
    # own = RT own-direction regularity: None = alpha + 1 = p, 1 = p - 1 (config 3's
    # literal "C^3" wording)
    p, n_el = 2, 2
    cpen = univariate.c_pen(p)
    h = 1.0 / n_el
    sp = [_space(p + 1, p if own is None else own, n_el, True) if d == k else _space(p, p - 1, n_el, False)
          for d in range(3)]
    X, W = _grid([n_el] * 3, p + 3)
    _, G, n = _trivariate(sp, X)
    A = _a_hat(G, W, k)
    N = A.shape[0]
    ek = np.eye(3)[k]
    # sigma^ over the six faces: 2[C/h w.v - ((grad^s w) n).v - ((grad^s v) n).w]
    xg, wg = splines.element_quadrature(np.linspace(0, 1, n_el + 1), p + 3)
    for d in range(3):
        others = [e for e in range(3) if e != d]
        for side in (0.0, 1.0):
            nrm = np.zeros(3)
            nrm[d] = 1.0 if side == 1.0 else -1.0
            pts = np.zeros((len(xg) ** 2, 3))
            wts = np.zeros(len(xg) ** 2)
            for a, (u, v) in enumerate(itertools.product(range(len(xg)), range(len(xg)))):
                pts[a, d] = side
                pts[a, others[0]] = xg[u]
                pts[a, others[1]] = xg[v]
                wts[a] = wg[u] * wg[v]
            Bf, Gf, _ = _trivariate(sp, pts)
            for q in range(len(wts)):
                Sn = []
                for i in range(N):
                    gw = np.outer(ek, Gf[q, i])
                    Sn.append(0.5 * (gw + gw.T) @ nrm)
                Sn = np.array(Sn)            # (N, 3): (grad^s w_i) n
                wv = np.outer(Bf[q], Bf[q])  # w_i . v_j = B_i B_j (both along e_k)
                cons = np.outer(Sn @ ek, Bf[q])  # ((grad^s w_i) n) . v_j
                A += wts[q] * 2.0 * (cpen / h * wv - cons - cons.T)
    Kn, Mn = univariate.rt_normal_pencil(p, n_el, own)
    Kt, Mt = univariate.rt_tangential_pencil(p, n_el)
    Ks = [Kn if d == k else Kt for d in range(3)]
    Ms = [Mn if d == k else Mt for d in range(3)]
    R = fd.assemble_R(Ks, Ms, [1.0 + (d == k) for d in range(3)])
    assert A.shape == R.shape
    assert np.max(np.abs(A - R)) < 1e-12 * np.max(np.abs(R))


def test_pressure_mass_equals_kronecker():
    p = 2
    n_els = (1, 2, 3)
    sp = [_space(p, p - 1, n, False) for n in n_els]
    X, W = _grid(n_els, p + 2)
    B, _, n = _trivariate(sp, X)
    Q = B.T @ (W[:, None] * B)      # [P_Q]_ij = int B_i B_j
    Mq = [univariate.pressure_mass(p, ne) for ne in n_els]
    PQ = kron.kron_dense(list(reversed(Mq)))  # M_3 (x) M_2 (x) M_1
    assert np.max(np.abs(Q - PQ)) < 1e-15 * 10
