"""GPU-resident preconditioned MINRES with a matrix-free Kronecker Stokes operator on the unit
cube / square ("making P_D-MINRES end-to-end on B200").

Operator (§3; identity map): a(w, v) = int 2 nu grad^s w : grad^s v gives
A_kk = sum_d c_d (K_d at d, M elsewhere) [+ Nitsche K~ for the RT tangential factors, P:701-704]
and, for r != s, A_rs = (G at s, G^T-type at r, M elsewhere) with G = int b'_test b_trial;
B_r = -( D^QV at r, M^QV elsewhere ), b(v, q) = -int q div v. Every block is a libfdp KronOp
(rectangular DMMA mode contractions with an accumulating epilogue); the 1D factors come from
libfdp's own quadrature (iga_mixed / iga_univariate). A separable viscosity
nu = sum_t c_t prod_d w_t(x_d) enters as extra weighted Kronecker terms; it must equal 1 on the
boundary so the Nitsche terms keep weight 1 (true for config 3's nu).

MINRES is Paige & Saunders' recurrence (tolerance 1e-8, x0 = 0) with every
vector operation in libfdp kernels (fdp_vec_dot / fdp_vec_lincomb); only the scalar recurrence
runs on the host. Stopping rule: preconditioned residual phibar_k / phibar_0 <= tol (C-15).

GMRES (NEXT-2, for the block-triangular P_T and constrained P_C) is full,
left-preconditioned GMRES (G-1) with the Arnoldi basis on the device; the
orthogonalization is classical Gram-Schmidt applied twice (two fdp_vec_multidot + fdp_vec_gemv
launch pairs instead of j dependent dot/axpy pairs per step; G-2), the small Hessenberg
least-squares problem by Givens rotations on the host.
"""
from __future__ import annotations

import math

import numpy as np

from . import (FDP_IGA_INTERIOR, FDP_IGA_NITSCHE, KronOp, iga_mass_diag_factor, iga_mixed,
               iga_quadrature, iga_univariate, minres_scalars, vec_dot, vec_gemv, vec_lincomb,
               vec_lincomb_dev, vec_multidot)


def _spaces(D, disc, p, rt_own_alpha=None):
    a = p - 1
    Q = (p, a, 0)
    if disc == "TH":
        V = [[(p + 1, a, FDP_IGA_INTERIOR)] * D for _ in range(D)]
    elif disc == "RT":
        N = (p + 1, a + 1 if rt_own_alpha is None else rt_own_alpha, FDP_IGA_INTERIOR)
        T = (p, a, 0)
        V = [[N if d == k else T for d in range(D)] for k in range(D)]
    else:
        raise ValueError(disc)
    return V, Q


class _GroupedOperator:
    """y = calA x for a block operator given as (KronOp, input block, output block) triples:
    applied by ONE kron_ops_apply call (all terms grouped per mode, one sum per output block),
    captured once per (x, y) pair into a CUDA graph and replayed."""

    def _finalize(self, group, sizes, device):
        import torch
        self.torch = torch
        self._group = group
        self.sizes = [int(v) for v in sizes]
        self.off_idx = np.concatenate([[0], np.cumsum(self.sizes)]).astype(np.int64)
        self.n = int(self.off_idx[-1])
        ops = [g[0] for g in group]
        self.ws = torch.empty(max(op.workspace_bytes(1) for op in ops) // 8 + 1, dtype=torch.float64,
                              device=f"cuda:{device}")
        self.gws = torch.empty(KronOp.group_workspace_bytes(ops) // 8 + 1, dtype=torch.float64,
                               device=f"cuda:{device}")
        self.grouped = True

    def apply(self, x, y):
        """y = calA x (graph-replayed; no allocation or host synchronisation inside)."""
        torch = self.torch
        key = (x.data_ptr(), y.data_ptr())
        if not hasattr(self, "_graphs"):
            self._graphs = {}
        g = self._graphs.get(key)
        if g is None:
            self._apply_direct(x, y)  # warm (kernel attributes, lazy module state)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._apply_direct(x, y)
            self._graphs[key] = g
        g.replay()
        return y

    def _apply_direct(self, x, y):
        o = self.off_idx
        blk = lambda v, k: v[o[k]:o[k + 1]]
        if self.grouped:
            KronOp.apply_group([g[0] for g in self._group], [blk(x, g[1]) for g in self._group],
                               [blk(y, g[2]) for g in self._group], [1.0] * len(self._group), 0.0,
                               self.gws)
            return y
        seen = set()
        for op, i, j in self._group:          # one kron_op_apply per block (reference path)
            op.apply(blk(x, i), blk(y, j), 1.0, 1.0 if j in seen else 0.0, self.ws)
            seen.add(j)
        return y


class StokesOperator(_GroupedOperator):
    """y = calA x for x = [u_1 | .. | u_D | p] (vec order, i1 fastest), on cuda:device."""

    def __init__(self, D: int, disc: str, p: int, n_el: int, nu_terms=None, device: int = 0,
                 rt_own_alpha=None):
        # rt_own_alpha: RT own-direction regularity (default p, the paper; p - 1 = config 3's
        # literal "C^3" wording, C-3)
        self.D = D
        nu_terms = nu_terms or [(1.0, None)]
        weighted = any(w is not None for _, w in nu_terms)
        q = p + 3 + (4 if weighted else 0)
        V, Qs = _spaces(D, disc, p, rt_own_alpha)
        xq, _ = iga_quadrature(n_el, q)
        mixed = lambda t, r, dt=0, dr=0, w=None: iga_mixed(t, r, n_el, dt, dr, q, None if w is None else w(xq))
        cp = 5.0 * p
        self.diag, self.off, self.B, self.BT = [], {}, [], []
        for k in range(D):
            terms, coef = [], []
            for ct, ws in nu_terms:
                wd = (lambda d: None) if ws is None else (lambda d, ws=ws: ws[d])
                Ms = [mixed(V[k][d], V[k][d], w=wd(d)) for d in range(D)]
                Ks = []
                for d in range(D):
                    if disc == "RT" and d != k and ws is None:
                        Kt, _ = iga_univariate(p, p - 1, n_el, FDP_IGA_NITSCHE, cp)
                        Ks.append(Kt)
                    else:
                        Ks.append(mixed(V[k][d], V[k][d], 1, 1, wd(d)))
                for d in range(D):
                    terms.append([Ks[e] if e == d else Ms[e] for e in range(D)])
                    coef.append(ct * (1.0 + (d == k)))
            self.diag.append(KronOp(terms, coef, device))
        for r in range(D):
            for s in range(D):
                if r == s:
                    continue
                terms, coef = [], []
                for ct, ws in nu_terms:
                    F = [mixed(V[r][d], V[s][d], int(d == s), int(d == r), None if ws is None else ws[d])
                         for d in range(D)]
                    terms.append(F)
                    coef.append(ct)
                self.off[(r, s)] = KronOp(terms, coef, device)
        for r in range(D):
            F = [mixed(Qs, V[r][d], 0, int(d == r)) for d in range(D)]
            self.B.append(KronOp([F], [-1.0], device))
            self.BT.append(KronOp([[np.asfortranarray(f.T) for f in F]], [-1.0], device))
        self.vel_dims = [self.diag[k].nin for k in range(D)]
        self.q_dims = self.B[0].nout
        group = []
        for r in range(D):
            group.append((self.diag[r], r, r))
            for s in range(D):
                if s != r:
                    group.append((self.off[(r, s)], s, r))
            group.append((self.BT[r], D, r))
        for r in range(D):
            group.append((self.B[r], r, D))
        sizes = [int(np.prod(v)) for v in self.vel_dims] + [int(np.prod(self.q_dims))]
        self._finalize(group, sizes, device)


_BUFFERS = {}


def minres(apply_A, apply_P, b, tol: float = 1e-8, maxit: int = 20000):
    """GPU MINRES: b (cuda float64), apply_A(x, y) / apply_P(r, z) write into y / z.
    Returns (x, iterations, history of phibar/beta1)."""
    import torch
    n = b.numel()
    dev = b.device
    # persistent buffers per (n, device): repeated solves hit the operator / preconditioner graph
    # caches (they are keyed by buffer addresses)
    key = (n, str(dev))
    if key not in _BUFFERS:
        _BUFFERS[key] = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(8)] + \
                        [torch.empty(2, dtype=torch.float64, device=dev)]
    x, r1, r2, y, v, w, w1, w2, dbuf = _BUFFERS[key]
    for t in (x, y, v, w, w1, w2):
        t.zero_()
    r1.copy_(b)
    r2.copy_(b)

    def dot(a, c, slot=0):
        vec_dot(a, c, dbuf[slot:slot + 1])
        return float(dbuf[slot].item())

    apply_P(r1, y)
    beta1 = dot(r1, y)
    if beta1 < 0:
        raise ValueError("preconditioner is not positive definite")
    beta1 = math.sqrt(beta1)
    if beta1 == 0.0:
        return x.clone(), 0, [0.0]
    oldb, beta, dbar, epsln, phibar = 0.0, beta1, 0.0, 0.0, beta1
    cs, sn = -1.0, 0.0
    hist = [1.0]
    eps = np.finfo(np.float64).eps
    for itn in range(1, maxit + 1):
        vec_lincomb(1.0 / beta, y, 0.0, None, 0.0, None, v)           # v = y / beta
        apply_A(v, y)                                                  # y = A v
        if itn >= 2:
            vec_lincomb(1.0, y, -beta / oldb, r1, 0.0, None, y)       # y -= (beta/oldb) r1
        alfa = dot(v, y)
        vec_lincomb(1.0, y, -alfa / beta, r2, 0.0, None, y)           # y -= (alfa/beta) r2
        r1, r2 = r2, r1
        r2.copy_(y)                                                     # r1 <- r2, r2 <- y
        apply_P(r2, y)
        oldb = beta
        beta = dot(r2, y)
        if beta < 0:
            raise ValueError("preconditioner is not positive definite")
        beta = math.sqrt(beta)
        oldeps = epsln
        delta = cs * dbar + sn * alfa
        gbar = sn * dbar - cs * alfa
        epsln = sn * beta
        dbar = -cs * beta
        gamma = max(math.hypot(gbar, beta), eps)
        cs = gbar / gamma
        sn = beta / gamma
        phi = cs * phibar
        phibar = sn * phibar
        w1, w2, w = w2, w, w1                                          # rotate buffers
        vec_lincomb(1.0 / gamma, v, -oldeps / gamma, w1, -delta / gamma, w2, w)
        vec_lincomb(1.0, x, phi, w, 0.0, None, x)
        hist.append(phibar / beta1)
        if phibar / beta1 <= tol:
            return x.clone(), itn, hist
    return x.clone(), maxit, hist


def nu_scalings_paper(gd, op: "StokesOperator", nu, q: int, device: int = 0):
    """Config 3's P^G scalings under the paper's definition (§6, DESIGN.md
    C-6b): D_V = diag(A_kk) / diag(P_V,k) with A_kk the nu-weighted velocity block of ``op``
    (kron_op_diagonal) and P_V,k the plain pencils; D_Q = diag(Q) / diag(P_Q) with
    Q = int nu^{-1} rho_i rho_j: libfdp's diagonal-of-mass factors contracted with
    nu^{-1} sampled on the q-point element Gauss grid by a KronOp on the GPU. Returns host arrays
    (D_V over all components, D_Q)."""
    import torch
    D = gd.D
    dv = []
    for k in range(D):
        dA = op.diag[k].diagonal()
        terms = [[gd.Ks[k][e] if e == d else gd.Ms[k][e] for e in range(D)] for d in range(D)]
        dP = KronOp(terms, gd.coef[k], device).diagonal()
        dv.append(dA / dP)
    F = iga_mass_diag_factor((gd.p, gd.p - 1, 0), gd.n_el, q)        # (n_q, points)
    xq, _ = iga_quadrature(gd.n_el, q)
    G = np.meshgrid(*([xq] * D), indexing="ij")
    w = torch.from_numpy(np.reshape(1.0 / nu(*G), -1, order="F")).to(f"cuda:{device}")
    Kq = KronOp([[F] * D], [1.0], device)
    dQ = torch.empty(int(np.prod(Kq.nout)), dtype=torch.float64, device=w.device)
    Kq.apply(w, dQ)
    dPq = KronOp([list(gd.Mq)], [1.0], device).diagonal()
    return np.concatenate(dv), dQ.cpu().numpy() / dPq


_DEV_MINRES = {}


def _fid(f):
    """Cache-key part of a callable: bound methods are new objects on every attribute access, so
    key them by (instance, function)."""
    return (id(getattr(f, "__self__", f)), getattr(getattr(f, "__func__", f), "__qualname__", ""))


def _refs(*fs):
    """Strong references to the callables' owners (and functions), kept in a cached graph's entry:
    while an entry lives its owners cannot be collected, so their ids cannot be reused."""
    return tuple((getattr(f, "__self__", f), getattr(f, "__func__", f)) for f in fs)


def _same_callables(ent, *fs):
    return all(o is getattr(f, "__self__", f) and fn is getattr(f, "__func__", f)
               for (o, fn), f in zip(ent["refs"], fs))


def minres_device(apply_A, apply_P, b, tol: float = 1e-8, maxit: int = 20000, unroll: int = 6):
    """MINRES with the scalar recurrence on the GPU (fdp_minres_scalars): `unroll` whole
    iterations (operator, preconditioner, dots, recurrence, vector updates) are captured into one
    CUDA graph and replayed; the host reads the `done` flag once per replay. The same arithmetic
    and stopping rule as ``minres``; iterations after convergence leave x untouched (their
    coefficients are 0), so the result and the reported count are exactly those of the
    converged step. apply_A / apply_P must be capturable (direct launches, no inner graph
    replay). unroll is a multiple of 6 so the r (period 2) and w (period 3) buffer rotations of
    the recurrence return to the captured roles. Returns (x, iterations, history)."""
    import torch
    assert unroll % 6 == 0
    n = b.numel()
    dev = b.device
    # bound methods are new objects on every attribute access: key them by (instance, function)
    key = (n, str(dev), unroll, _fid(apply_A), _fid(apply_P))
    ent = _DEV_MINRES.get(key)
    if ent is not None and not _same_callables(ent, apply_A, apply_P):
        ent = None  # an id reused by a new object: the cached graph belongs to the old one
    if ent is None:
        _DEV_MINRES.clear()
        vecs = [torch.zeros(n, dtype=torch.float64, device=dev) for _ in range(8)]
        state = torch.zeros(32, dtype=torch.float64, device=dev)
        hist = torch.zeros(maxit + 1, dtype=torch.float64, device=dev)
        ent = {"vecs": vecs, "state": state, "hist": hist, "graph": None,
               "refs": _refs(apply_A, apply_P)}
        _DEV_MINRES[key] = ent
    x, r1, r2, y, v, w, w1, w2 = ent["vecs"]
    state, hist = ent["state"], ent["hist"]
    if hist.numel() < maxit + 1:
        hist = ent["hist"] = torch.zeros(maxit + 1, dtype=torch.float64, device=dev)
        ent["graph"] = None
    def init():
        for t in (x, w, w1, w2):
            t.zero_()
        r1.copy_(b)
        r2.copy_(b)
        apply_P(r1, y)
        state.zero_()
        state[13] = tol
        vec_dot(r1, y, state[9:10])
        minres_scalars(0, state)

    init()
    kv, ky1, ky2, kw, kx = (state[16:19], state[19:22], state[22:25], state[25:28], state[28:31])

    def iterations():
        R1, R2, W, W1, W2 = r1, r2, w, w1, w2
        for _ in range(unroll):
            minres_scalars(1, state)
            vec_lincomb_dev(kv, y, None, None, v)           # v = y / beta
            apply_A(v, y)                                   # y = A v
            vec_lincomb_dev(ky1, y, R1, None, y)            # y -= (beta/oldb) r1
            vec_dot(v, y, state[8:9])                       # alfa
            minres_scalars(2, state)
            vec_lincomb_dev(ky2, y, R2, None, y)            # y -= (alfa/beta) r2
            R1, R2 = R2, R1
            R2.copy_(y)
            apply_P(R2, y)
            vec_dot(R2, y, state[9:10])                     # beta^2
            minres_scalars(3, state, hist)
            W1, W2, W = W2, W, W1
            vec_lincomb_dev(kw, v, W1, W2, W)               # w = (v - oldeps w1 - delta w2) / gamma
            vec_lincomb_dev(kx, x, W, None, x)              # x += phi w

    if ent["graph"] is None:
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):  # warm-up (advances the recurrence: re-initialised below)
            iterations()
        torch.cuda.current_stream().wait_stream(s)
        with torch.cuda.graph(g):
            iterations()
        ent["graph"] = g
        init()
    g = ent["graph"]
    while True:
        g.replay()
        st = state[10:13].tolist()   # itn, done, itn_done (the one host read per replay)
        if st[1] != 0.0 or st[0] >= maxit:
            break
    if state[14].item() != 0.0:
        raise ValueError("preconditioner is not positive definite")
    its = int(st[2]) if st[1] != 0.0 else maxit
    h = [1.0] + hist[1:its + 1].tolist()
    return x.clone(), its, h


_GM_BUFFERS = {}


def gmres(apply_A, apply_P, b, tol: float = 1e-8, maxit: int = 500):
    """GPU GMRES for A x = b with left preconditioner P: apply_A(x, y) / apply_P(r, z) write into
    y / z. Stops when ||P^{-1}(b - A x_k)|| / ||P^{-1} b|| <= tol. Returns (x, iterations, history).

    apply_A / apply_P are always called on the same two fixed buffers (so their CUDA graphs,
    keyed by buffer addresses, are captured once)."""
    import torch
    n = b.numel()
    dev = b.device
    m = min(maxit, n)
    key = (n, m, str(dev))
    if key not in _GM_BUFFERS:
        V = torch.empty((m + 1, n), dtype=torch.float64, device=dev)
        vin = torch.empty(n, dtype=torch.float64, device=dev)
        t = torch.empty(n, dtype=torch.float64, device=dev)
        w = torch.empty(n, dtype=torch.float64, device=dev)
        h = torch.empty(2 * (m + 1) + 1, dtype=torch.float64, device=dev)
        from . import lib
        ws = torch.empty(max(1, int(lib.fdp_vec_multidot_workspace_bytes(m + 1)) // 8),
                         dtype=torch.float64, device=dev)
        _GM_BUFFERS.clear()
        _GM_BUFFERS[key] = (V, vin, t, w, h, ws)
    V, vin, t, w, h, ws = _GM_BUFFERS[key]
    vin.copy_(b)
    apply_P(vin, w)
    vec_dot(w, w, h[0:1])
    beta = math.sqrt(float(h[0].item()))
    if beta == 0.0:
        return torch.zeros_like(b), 0, [0.0]
    vec_lincomb(1.0 / beta, w, 0.0, None, 0.0, None, V[0])
    H = np.zeros((m + 1, m))
    cs = np.zeros(m)
    sn = np.zeros(m)
    g = np.zeros(m + 1)
    g[0] = beta
    hist = [1.0]
    k = 0
    h1, h2, nrm = h[:m + 1], h[m + 1:2 * m + 2], h[2 * m + 2:]
    for j in range(m):
        vin.copy_(V[j])
        apply_A(vin, t)
        apply_P(t, w)                                            # w = P^{-1} A v_j
        vec_multidot(V, j + 1, w, h1, ws)                        # CGS, pass 1
        vec_gemv(V, j + 1, h1, -1.0, w, 1.0)
        vec_multidot(V, j + 1, w, h2, ws)                        # CGS, pass 2
        vec_gemv(V, j + 1, h2, -1.0, w, 1.0)
        vec_dot(w, w, nrm)
        hh = h.cpu().numpy()                                     # the one host sync per step
        H[:j + 1, j] = hh[:j + 1] + hh[m + 1:m + 2 + j]
        H[j + 1, j] = math.sqrt(hh[2 * m + 2])
        if H[j + 1, j] != 0.0:
            vec_lincomb(1.0 / H[j + 1, j], w, 0.0, None, 0.0, None, V[j + 1])
        for i in range(j):                                       # previous rotations
            tmp = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
            H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
            H[i, j] = tmp
        den = math.hypot(H[j, j], H[j + 1, j])
        cs[j] = H[j, j] / den
        sn[j] = H[j + 1, j] / den
        H[j, j] = den
        H[j + 1, j] = 0.0
        g[j + 1] = -sn[j] * g[j]
        g[j] = cs[j] * g[j]
        k = j + 1
        hist.append(abs(g[j + 1]) / beta)
        if abs(g[j + 1]) / beta <= tol or H[j, j] == 0.0:
            break
    y = np.zeros(k)
    for i in range(k - 1, -1, -1):
        y[i] = (g[i] - H[i, i + 1:k] @ y[i + 1:k]) / H[i, i]
    h1[:k].copy_(torch.from_numpy(y))
    x = torch.empty_like(b)
    vec_gemv(V, k, h1, 1.0, x, 0.0)
    return x, k, hist


_DEV_GMRES = {}


def gmres_device(apply_A, apply_P, b, tol: float = 1e-8, maxit: int = 500, unroll: int = 4):
    """GMRES with the Arnoldi bookkeeping on the GPU (fdp_gmres_scalars; basis indices and counts
    read from device memory by fdp_vec_copy_indexed / _store_indexed / _multidot_dev /
    _gemv_dev): `unroll` whole steps are one CUDA graph, the host reads the `done` flag once per
    replay. Same arithmetic and stopping rule as ``gmres`` (classical Gram-Schmidt twice, Givens
    rotations); steps after convergence change nothing. apply_A / apply_P must be capturable
    (direct launches). Returns (x, iterations, history)."""
    import ctypes

    import torch
    from . import _check, lib
    n = b.numel()
    dev = b.device
    m = min(maxit, n)
    key = (n, m, str(dev), unroll, _fid(apply_A), _fid(apply_P))
    ent = _DEV_GMRES.get(key)
    if ent is not None and not _same_callables(ent, apply_A, apply_P):
        ent = None
    st = lambda: torch.cuda.current_stream().cuda_stream
    if ent is None:
        _DEV_GMRES.clear()
        f64 = dict(dtype=torch.float64, device=dev)
        ent = {
            "V": torch.empty((m + 1, n), **f64), "vin": torch.empty(n, **f64), "t": torch.empty(n, **f64),
            "w": torch.empty(n, **f64), "h1": torch.zeros(m + 1, **f64), "h2": torch.zeros(m + 1, **f64),
            "H": torch.zeros((m, m + 1), **f64), "hist": torch.zeros(m + 1, **f64),
            "ds": torch.zeros(8 + 3 * (m + 1), **f64),
            "is": torch.zeros(5, dtype=torch.int32, device=dev),
            "scr": torch.empty(max(1, int(lib.fdp_vec_multidot_workspace_bytes(m + 1)) // 8), **f64),
            "graph": None,
            "refs": _refs(apply_A, apply_P),
        }
        _DEV_GMRES[key] = ent
    V, vin, t, w = ent["V"], ent["vin"], ent["t"], ent["w"]
    h1, h2, H, hist, ds, is_, scr = ent["h1"], ent["h2"], ent["H"], ent["hist"], ent["ds"], ent["is"], ent["scr"]
    P = lambda x: ctypes.c_void_p(x.data_ptr())
    ldv = V.stride(0)

    def scalars(phase):
        _check(lib.fdp_gmres_scalars(phase, P(is_), P(ds), P(H), m + 1, P(h1), P(h2), P(hist), m, st()))

    def store():  # V[istate[4]] = dstate[2] * w
        _check(lib.fdp_vec_store_indexed(P(V), ldv, ctypes.c_void_p(is_.data_ptr() + 16), P(w),
                                         ctypes.c_void_p(ds.data_ptr() + 16), n, st()))

    def steps():
        for _ in range(unroll):
            _check(lib.fdp_vec_copy_indexed(P(V), ldv, P(is_), P(vin), n, st()))
            apply_A(vin, t)
            apply_P(t, w)                                              # w = P^{-1} A v_j
            mc = ctypes.c_void_p(is_.data_ptr() + 12)                  # j + 1
            for h in (h1, h2):                                         # classical GS, twice
                _check(lib.fdp_vec_multidot_dev(P(V), ldv, mc, m + 1, P(w), n, P(h), P(scr), st()))
                _check(lib.fdp_vec_gemv_dev(P(V), ldv, mc, m + 1, P(h), -1.0, P(w), 1.0, n, st()))
            vec_dot(w, w, ds[3:4])
            scalars(1)
            store()

    def init():
        vin.copy_(b)
        apply_P(vin, w)
        ds.zero_()
        ds[1] = tol
        vec_dot(w, w, ds[4:5])
        scalars(0)
        store()

    init()
    if ent["graph"] is None:
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # warm-up (advances the iteration: re-initialised below)
            steps()
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            steps()
        ent["graph"] = g
        init()
    g = ent["graph"]
    while True:
        g.replay()
        iv = is_.tolist()                                              # the one host read per replay
        if iv[1] or iv[0] >= m:
            break
    k = iv[2] if iv[1] else m
    if k == 0:
        return torch.zeros_like(b), 0, [0.0]
    R = H[:k, :k].cpu().numpy().T                                      # R[i, j] = H column j, row i
    gv = ds[8 + 2 * (m + 1): 8 + 2 * (m + 1) + k].cpu().numpy()
    y = np.zeros(k)
    for i in range(k - 1, -1, -1):
        y[i] = (gv[i] - R[i, i + 1:k] @ y[i + 1:k]) / R[i, i]
    h1[:k].copy_(torch.from_numpy(y))
    x = torch.empty_like(b)
    vec_gemv(V, k, h1, 1.0, x, 0.0)
    return x, k, [1.0] + hist[1:k + 1].tolist()
