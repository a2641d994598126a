"""Python binding of libfdp (include/fdp.h): argument marshalling only.

Every step of the preconditioner application runs in libfdp's sm_100a kernels; torch provides
device memory and streams. There is no CPU fallback: if ``libfdp.so`` is missing or a call fails
the binding raises. Names follow the C ABI (``fd_setup`` -> :class:`FD`, ``kron_mass_*`` ->
:class:`KronMass`, ``block_precond_*`` -> :class:`BlockPrecond`).

Paper: Montardini, Sangalli, Tani, arXiv:1712.00403. Citations P:L are its lines.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

__all__ = ["FdpError", "lib", "iga_univariate", "iga_greville", "gen_eig", "FD", "KronMass",
           "BlockPrecond", "Discretization", "discretization", "nu_scalings", "LIB_PATH"]

LIB_PATH = os.environ.get("FDP_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                           "libfdp.so")

FDP_IGA_INTERIOR = 1
FDP_IGA_NITSCHE = 2
FDP_MASS_INVERSE = 0
FDP_MASS_FORWARD = 1

_c_double_p = ctypes.POINTER(ctypes.c_double)
_c_int32_p = ctypes.POINTER(ctypes.c_int32)


class FdpError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{_status_name(status)}: {message}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libfdp.so not built at {LIB_PATH}: run `make` or __graft_entry__.build()")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, i32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
    sig = {
        "fdp_status_string": (ctypes.c_char_p, [i32]),
        "fdp_last_error": (ctypes.c_char_p, []),
        "fdp_version": (ctypes.c_char_p, []),
        "iga_univariate": (i32, [i32, i32, i32, i32, ctypes.c_double, i32, vp, vp, _c_int32_p]),
        "iga_greville": (i32, [i32, i32, i32, i32, vp, _c_int32_p]),
        "fdp_gen_eig": (i32, [i32, vp, vp, vp, vp]),
        "fdp_kron_diag": (i32, [i32, vp, i32, vp, vp, i32, vp]),
        "fd_setup": (i32, [i32, vp, vp, vp, vp, i32, i64, ctypes.POINTER(vp)]),
        "fd_get_eigs": (i32, [vp, i32, vp, vp]),
        "fd_size": (i64, [vp]),
        "fd_workspace_bytes": (sz, [vp, i64]),
        "fd_apply": (i32, [vp, vp, vp, vp, i64, vp, vp]),
        "fd_destroy": (i32, [vp]),
        "kron_mass_setup": (i32, [i32, vp, vp, i32, ctypes.POINTER(vp)]),
        "kron_mass_size": (i64, [vp]),
        "kron_mass_apply": (i32, [vp, i32, vp, vp, vp, i64, vp]),
        "kron_mass_destroy": (i32, [vp]),
        "block_precond_setup": (i32, [i32, vp, vp, vp, vp, ctypes.POINTER(vp)]),
        "block_precond_size": (i64, [vp]),
        "block_precond_workspace_bytes": (sz, [vp, i64]),
        "block_precond_apply": (i32, [vp, vp, vp, i64, vp, vp]),
        "block_precond_apply_host": (i32, [vp, vp, vp, i64, vp]),
        "block_precond_destroy": (i32, [vp]),
        "fdp_block_launch_count": (i32, [vp, i64]),
        "fdp_debug_k1_launches": (i64, [i32]),
        "block_precond_profile": (i32, [vp, i32]),
        "fdp_slab_range": (i32, [i64, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]),
        "kron_op_setup": (i32, [i32, i32, vp, vp, vp, vp, i32, ctypes.POINTER(vp)]),
        "kron_op_workspace_bytes": (sz, [vp, i64]),
        "kron_op_apply": (i32, [vp, vp, i64, vp, i64, ctypes.c_double, ctypes.c_double, i64, vp, vp]),
        "kron_op_destroy": (i32, [vp]),
        "kron_ops_workspace_bytes": (sz, [i32, ctypes.POINTER(vp)]),
        "block_tri_workspace_bytes": (sz, [vp, i32, ctypes.POINTER(vp), ctypes.POINTER(vp)]),
        "block_tri_apply": (i32, [vp, i32, ctypes.POINTER(vp), ctypes.POINTER(vp), vp, vp, vp, vp]),
        "iga_geometry_coeffs": (i32, [i32, i32, i32, i32, vp, vp]),
        "iga_separable_fit": (i32, [i32, vp, ctypes.POINTER(vp), i32, ctypes.c_double, vp, vp, vp]),
        "fd_operator_diagonal": (i32, [vp, vp]),
        "kron_op_diagonal": (i32, [vp, vp]),
        "iga_mass_diag_factor": (i32, [i32, i32, i32, i32, i32, vp, ctypes.POINTER(ctypes.c_int32)]),
        "fdp_vec_lincomb_dev": (i32, [vp, vp, vp, vp, vp, i64, vp]),
        "fdp_minres_scalars": (i32, [i32, vp, vp, i32, vp]),
        "fdp_vec_copy_indexed": (i32, [vp, i64, vp, vp, i64, vp]),
        "fdp_vec_store_indexed": (i32, [vp, i64, vp, vp, vp, i64, vp]),
        "fdp_vec_multidot_dev": (i32, [vp, i64, vp, i32, vp, i64, vp, vp, vp]),
        "fdp_vec_gemv_dev": (i32, [vp, i64, vp, i32, vp, ctypes.c_double, vp, ctypes.c_double, i64, vp]),
        "fdp_gmres_scalars": (i32, [i32, vp, vp, vp, i32, vp, vp, vp, i32, vp]),
        "fdp_host_alloc": (vp, [sz]),
        "fdp_host_free": (i32, [vp]),
        "fdp_vec_multidot_workspace_bytes": (sz, [i32]),
        "fdp_vec_multidot": (i32, [vp, i64, i32, vp, i64, vp, vp, vp]),
        "fdp_vec_gemv": (i32, [vp, i64, i32, vp, ctypes.c_double, vp, ctypes.c_double, i64, vp]),
        "kron_ops_apply": (i32, [i32, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp),
                                 ctypes.POINTER(ctypes.c_double), ctypes.c_double, vp, vp]),
        "iga_quadrature": (i32, [i32, i32, vp, vp]),
        "iga_mixed": (i32, [i32, i32, i32, i32, i32, i32, i32, i32, i32, i32, vp, vp, _c_int32_p, _c_int32_p]),
        "fdp_vec_dot": (i32, [vp, vp, i64, vp, vp]),
        "fdp_vec_lincomb": (i32, [ctypes.c_double, vp, ctypes.c_double, vp, ctypes.c_double, vp, vp, i64, vp]),
        "fd_slab_workspace_bytes": (sz, [vp, i32, i32]),
        "fd_apply_slab": (i32, [vp, i32, i32, i32, vp, vp, vp, vp, vp]),
        "fd_apply_slab_peer": (i32, [vp, i32, i32, i32, vp, vp, vp, vp, vp, vp]),
        "kron_mass_apply_slab_peer": (i32, [vp, i32, i32, i32, vp, vp, vp, vp, vp, vp]),
        "fdp_peer_barrier": (i32, [vp, vp, i32, i32, vp]),
        "fdp_comm_blob_bytes": (sz, [vp, i32]),
        "fdp_comm_create": (i32, [vp, i32, i32, ctypes.POINTER(vp), vp]),
        "fdp_comm_connect": (i32, [vp, vp]),
        "block_precond_sharded_size": (i64, [vp, i32, i32]),
        "block_precond_sharded_workspace_bytes": (sz, [vp, vp]),
        "block_precond_apply_sharded": (i32, [vp, vp, vp, vp, vp, vp]),
        "fdp_comm_destroy": (i32, [vp]),
        "fdp_nccl_unique_id": (i32, [vp]),
        "fdp_slab_exchange_counts": (i32, [vp, i32, i32, i32, vp, vp]),
        "fdp_comm_init": (i32, [i32, i32, vp, i32, ctypes.POINTER(vp)]),
        "fd_sharded_workspace_bytes": (sz, [vp, vp]),
        "fd_apply_sharded": (i32, [vp, vp, vp, vp, vp, vp, vp]),
        "fdp_peer_alloc": (i32, [sz, i32, ctypes.POINTER(vp), vp]),
        "fdp_peer_open": (i32, [vp, i32, ctypes.POINTER(vp)]),
        "fdp_peer_close": (i32, [vp]),
        "fdp_peer_free": (i32, [vp]),
        "kron_mass_slab_workspace_bytes": (sz, [vp, i32, i32]),
        "kron_mass_apply_slab": (i32, [vp, i32, i32, i32, vp, vp, vp, vp, vp]),
        "block_precond_profile_read": (i32, [vp, i32, vp, vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L


lib = _load()


def _status_name(s: int) -> str:
    return lib.fdp_status_string(s).decode()


def _check(status: int):
    if status != 0:
        raise FdpError(status, lib.fdp_last_error().decode())


def _host(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _fortran(a) -> np.ndarray:
    return np.asfortranarray(a, dtype=np.float64)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _dev(t, name: str, numel: int | None = None) -> int:
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name}: expected a torch.Tensor on CUDA")
    if t.dtype != torch.float64 or not t.is_cuda or not t.is_contiguous():
        raise TypeError(f"{name}: expected a contiguous float64 CUDA tensor")
    if numel is not None and t.numel() < numel:
        raise ValueError(f"{name}: needs {numel} elements, has {t.numel()}")
    return t.data_ptr()


def _stream(stream) -> int:
    import torch
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


# ----------------------------------------------------------------------------------------------
# host helpers
# ----------------------------------------------------------------------------------------------
def iga_univariate(deg: int, alpha: int, n_el: int, flags: int = 0, c_pen: float = 0.0, q: int = 0):
    """(K, M) of the univariate space built by libfdp (column-major)."""
    n = ctypes.c_int32(0)
    _check(lib.iga_univariate(deg, alpha, n_el, flags, c_pen, q, None, None, ctypes.byref(n)))
    K = np.zeros((n.value, n.value), order="F")
    M = np.zeros((n.value, n.value), order="F")
    _check(lib.iga_univariate(deg, alpha, n_el, flags, c_pen, q, _ptr(K), _ptr(M), ctypes.byref(n)))
    return K, M


def iga_greville(deg: int, alpha: int, n_el: int, flags: int = 0) -> np.ndarray:
    n = ctypes.c_int32(0)
    _check(lib.iga_greville(deg, alpha, n_el, flags, None, ctypes.byref(n)))
    g = np.zeros(n.value)
    _check(lib.iga_greville(deg, alpha, n_el, flags, _ptr(g), ctypes.byref(n)))
    return g


def gen_eig(K, M):
    """Host generalized eigensolver of libfdp (Algorithm 1 step 1): (lambda, U)."""
    K, M = _fortran(K), _fortran(M)
    n = K.shape[0]
    U = np.zeros((n, n), order="F")
    lam = np.zeros(n)
    _check(lib.fdp_gen_eig(n, _ptr(K), _ptr(M), _ptr(U), _ptr(lam)))
    return lam, U


# ----------------------------------------------------------------------------------------------
# handles
# ----------------------------------------------------------------------------------------------
class FD:
    """fd_setup / fd_apply: x = dscale o U Lambda^{-1} U^T (dscale o b) (Algorithm 1)."""

    def __init__(self, Ks, Ms, coef, device: int = 0, max_batch: int = 0):
        D = len(Ks)
        self.D = D
        self.dims = [int(K.shape[0]) for K in Ks]
        self._K = [_fortran(K) for K in Ks]
        self._M = [_fortran(M) for M in Ms]
        n = (ctypes.c_int32 * D)(*self.dims)
        Kp = (ctypes.c_void_p * D)(*[k.ctypes.data for k in self._K])
        Mp = (ctypes.c_void_p * D)(*[m.ctypes.data for m in self._M])
        c = (ctypes.c_double * D)(*[float(x) for x in coef])
        h = ctypes.c_void_p()
        _check(lib.fd_setup(D, n, Kp, Mp, c, device, max_batch, ctypes.byref(h)))
        self.h = h
        self.N = int(lib.fd_size(h))
        self.device = device

    def workspace_bytes(self, batch: int) -> int:
        return int(lib.fd_workspace_bytes(self.h, batch))

    def operator_diagonal(self):
        """diag(sum_d coef_d (M_D (x) .. K_d .. (x) M_1)) (fd_operator_diagonal)."""
        out = np.zeros(self.N)
        _check(lib.fd_operator_diagonal(self.h, _ptr(out)))
        return out

    def get_eigs(self, d: int):
        n = self.dims[d]
        U = np.zeros((n, n), order="F")
        lam = np.zeros(n)
        _check(lib.fd_get_eigs(self.h, d, _ptr(U), _ptr(lam)))
        return lam, U

    def apply(self, b, x=None, dscale=None, batch: int = 1, workspace=None, stream=None):
        import torch
        if x is None:
            x = torch.empty_like(b)
        numel = self.N * batch
        wsn = max(1, self.workspace_bytes(batch) // 8)
        if workspace is None:
            workspace = torch.empty(wsn, dtype=torch.float64, device=b.device)
        ws = _dev(workspace, "workspace", wsn)
        _check(lib.fd_apply(self.h, _dev(b, "b", numel), _dev(x, "x", numel),
                            None if dscale is None else _dev(dscale, "dscale", self.N), batch, ws,
                            _stream(stream)))
        return x

    def close(self):
        if getattr(self, "h", None):
            lib.fd_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def iga_quadrature(n_el: int, q: int):
    """Gauss points / weights of libfdp's element quadrature on [0, 1] (n_el * q each)."""
    x = np.zeros(n_el * q)
    w = np.zeros(n_el * q)
    _check(lib.iga_quadrature(n_el, q, _ptr(x), _ptr(w)))
    return x, w


def iga_mass_diag_factor(space, n_el: int, q: int):
    """(n x n_el q) host matrix of w_g b_i(x_g)^2 at libfdp's element Gauss points;
    space = (deg, alpha, flags)."""
    deg, alpha, flags = space
    n = ctypes.c_int32(0)
    _check(lib.iga_mass_diag_factor(deg, alpha, n_el, flags, q, None, ctypes.byref(n)))
    out = np.zeros((n.value, n_el * q), order="F")
    _check(lib.iga_mass_diag_factor(deg, alpha, n_el, flags, q, _ptr(out), ctypes.byref(n)))
    return out


def iga_mixed(test, trial, n_el: int, dtest: int = 0, dtrial: int = 0, q: int = 0, wq=None):
    """int wt b_test^(dtest) b_trial^(dtrial); test/trial = (deg, alpha, flags)."""
    nt, nr = ctypes.c_int32(0), ctypes.c_int32(0)
    _check(lib.iga_mixed(*test, *trial, n_el, dtest, dtrial, q, None, None, ctypes.byref(nt), ctypes.byref(nr)))
    out = np.zeros((nt.value, nr.value), order="F")
    wq_ = None if wq is None else _host(wq)
    _check(lib.iga_mixed(*test, *trial, n_el, dtest, dtrial, q, None if wq_ is None else _ptr(wq_), _ptr(out),
                         ctypes.byref(nt), ctypes.byref(nr)))
    return out


class KronOp:
    """kron_op_*: y = beta y + alpha sum_t c_t (F_{t,D} (x) .. (x) F_{t,1}) x, rectangular factors."""

    def __init__(self, terms, coef, device: int = 0):
        D = len(terms[0])
        self.D = D
        self.nin = [int(F.shape[1]) for F in terms[0]]
        self.nout = [int(F.shape[0]) for F in terms[0]]
        self._F = [_fortran(F) for T in terms for F in T]
        self._coef = [float(x) for x in coef]
        nin = (ctypes.c_int32 * D)(*self.nin)
        nout = (ctypes.c_int32 * D)(*self.nout)
        Fp = (ctypes.c_void_p * len(self._F))(*[F.ctypes.data for F in self._F])
        c = (ctypes.c_double * len(coef))(*[float(x) for x in coef])
        h = ctypes.c_void_p()
        _check(lib.kron_op_setup(D, len(terms), nin, nout, Fp, c, device, ctypes.byref(h)))
        self.h = h
        self.device = device

    def workspace_bytes(self, batch: int = 1) -> int:
        return int(lib.kron_op_workspace_bytes(self.h, batch))

    def apply(self, x, y, alpha=1.0, beta=0.0, workspace=None, batch=1, xbs=0, ybs=0, stream=None):
        import torch
        if workspace is None:
            workspace = torch.empty(max(1, self.workspace_bytes(batch) // 8), dtype=torch.float64,
                                    device=x.device)
        _check(lib.kron_op_apply(self.h, _dev(x, "x"), xbs, _dev(y, "y"), ybs, alpha, beta, batch,
                                 _dev(workspace, "workspace"), _stream(stream)))
        return y

    def diagonal(self):
        """diag of a square operator (kron_op_diagonal)."""
        out = np.zeros(int(np.prod(self.nin)))
        _check(lib.kron_op_diagonal(self.h, _ptr(out)))
        return out

    @staticmethod
    def _handles(ops):
        return (ctypes.c_void_p * len(ops))(*[op.h.value for op in ops])

    @staticmethod
    def group_workspace_bytes(ops) -> int:
        return int(lib.kron_ops_workspace_bytes(len(ops), KronOp._handles(ops)))

    @staticmethod
    def apply_group(ops, xs, ys, alphas, beta=0.0, workspace=None, stream=None):
        """kron_ops_apply: for every distinct output Y among ys, Y = beta Y + sum alpha_i ops_i xs_i
        (batch 1), all terms as one grouped launch per mode plus one summation per output."""
        import torch
        n = len(ops)
        if workspace is None:
            workspace = torch.empty(max(1, KronOp.group_workspace_bytes(ops) // 8),
                                    dtype=torch.float64, device=xs[0].device)
        X = (ctypes.c_void_p * n)(*[_dev(x, "x") for x in xs])
        Y = (ctypes.c_void_p * n)(*[_dev(y, "y") for y in ys])
        A = (ctypes.c_double * n)(*[float(a) for a in alphas])
        _check(lib.kron_ops_apply(n, KronOp._handles(ops), X, Y, A, beta, _dev(workspace, "workspace"),
                                  _stream(stream)))

    def close(self):
        if getattr(self, "h", None):
            lib.kron_op_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def vec_dot(x, y, out, stream=None):
    _check(lib.fdp_vec_dot(_dev(x, "x"), _dev(y, "y"), x.numel(), _dev(out, "out"), _stream(stream)))
    return out


def vec_lincomb(a, x, b, y, c, z, out, stream=None):
    _check(lib.fdp_vec_lincomb(a, _dev(x, "x"), b, None if y is None else _dev(y, "y"), c,
                               None if z is None else _dev(z, "z"), _dev(out, "out"), out.numel(),
                               _stream(stream)))
    return out


def vec_lincomb_dev(k, x, y, z, out, stream=None):
    """out = k[0] x + k[1] y + k[2] z, k a 3-element cuda tensor (zero terms skipped)."""
    _check(lib.fdp_vec_lincomb_dev(_dev(k, "k"), _dev(x, "x"), None if y is None else _dev(y, "y"),
                                   None if z is None else _dev(z, "z"), _dev(out, "out"), out.numel(),
                                   _stream(stream)))
    return out


def minres_scalars(phase: int, state, hist=None, stream=None):
    """fdp_minres_scalars: the MINRES scalar recurrence on the device (state layout in fdp.h)."""
    _check(lib.fdp_minres_scalars(phase, _dev(state, "state"), None if hist is None else _dev(hist, "hist"),
                                  0 if hist is None else hist.numel(), _stream(stream)))


class _PinnedBuffer:
    def __init__(self, nbytes):
        self.ptr = lib.fdp_host_alloc(nbytes)
        if not self.ptr:
            raise FdpError(6, lib.fdp_last_error().decode())

    def __del__(self):
        try:
            lib.fdp_host_free(self.ptr)
        except Exception:
            pass


def host_empty(shape, dtype=np.float64) -> np.ndarray:
    """numpy array in page-locked host memory (fdp_host_alloc), freed with the array."""
    dt = np.dtype(dtype)
    n = int(np.prod(shape)) * dt.itemsize
    buf = _PinnedBuffer(max(n, 1))
    raw = (ctypes.c_char * max(n, 1)).from_address(buf.ptr)
    raw._fdp_pinned = buf  # the ctypes array (the numpy base) keeps the allocation alive
    arr = np.ctypeslib.as_array(raw)
    return arr[:n].view(dt).reshape(shape)


def vec_multidot(V, m, w, h, workspace=None, stream=None):
    """h[:m] = V[:m] @ w (fdp_vec_multidot; V a 2-D cuda tensor of row vectors)."""
    import torch
    if workspace is None:
        workspace = torch.empty(max(1, int(lib.fdp_vec_multidot_workspace_bytes(max(m, 1))) // 8),
                                dtype=torch.float64, device=w.device)
    _check(lib.fdp_vec_multidot(_dev(V, "V"), V.stride(0), m, _dev(w, "w"), w.numel(), _dev(h, "h"),
                                _dev(workspace, "workspace"), _stream(stream)))
    return h


def vec_gemv(V, m, h, alpha, w, beta, stream=None):
    """w = beta w + alpha V[:m]^T h[:m] (fdp_vec_gemv)."""
    _check(lib.fdp_vec_gemv(_dev(V, "V"), V.stride(0), m, _dev(h, "h"), alpha, _dev(w, "w"), beta,
                            w.numel(), _stream(stream)))
    return w


FDP_GEOM_IDENTITY = 0
FDP_GEOM_ANNULUS = 1


def iga_geometry_coeffs(kind: int, D: int, k: int, x):
    """c^k_dd of C_k^TH at the tensor grid of the 1D points x: list of D arrays, each shaped
    (len(x),) * D in vec order (i1 fastest) flattened (iga_geometry_coeffs)."""
    x = _host(x)
    nq = x.size
    out = np.zeros(D * nq ** D)
    _check(lib.iga_geometry_coeffs(kind, D, k, nq, _ptr(x), _ptr(out)))
    return [out[d * nq ** D:(d + 1) * nq ** D] for d in range(D)]


def iga_separable_fit(c, nq, max_sweeps: int = 50, tol: float = 1e-8):
    """(tau, mu, sweeps): per-direction node values of c_d ~ tau_d prod_{m != d} mu_m."""
    D = len(c)
    cs = [_host(ci) for ci in c]
    n = (ctypes.c_int32 * D)(*[int(v) for v in nq])
    cp = (ctypes.c_void_p * D)(*[ci.ctypes.data for ci in cs])
    tau = np.zeros(int(sum(nq)))
    mu = np.zeros(int(sum(nq)))
    sw = ctypes.c_int32(0)
    _check(lib.iga_separable_fit(D, n, cp, max_sweeps, tol, _ptr(tau), _ptr(mu), ctypes.byref(sw)))
    off = np.concatenate([[0], np.cumsum(nq)])
    return ([tau[off[d]:off[d + 1]] for d in range(D)], [mu[off[d]:off[d + 1]] for d in range(D)],
            sw.value)


def slab_range(n: int, nranks: int, rank: int):
    """(lo, len) of rank's share of an axis of length n (fdp_slab_range)."""
    lo, ln = ctypes.c_int64(), ctypes.c_int64()
    _check(lib.fdp_slab_range(n, nranks, rank, ctypes.byref(lo), ctypes.byref(ln)))
    return lo.value, ln.value


def slab_exchange_counts(dims, nranks: int, rank: int, exchange: int):
    """fdp_slab_exchange_counts: (send counts, recv counts) per peer of exchange 1 or 2."""
    d = np.ascontiguousarray(dims, dtype=np.int32)
    sc = np.zeros(nranks, dtype=np.int64)
    rc = np.zeros(nranks, dtype=np.int64)
    _check(lib.fdp_slab_exchange_counts(_ptr(d), nranks, rank, exchange, _ptr(sc), _ptr(rc)))
    return [int(v) for v in sc], [int(v) for v in rc]


def fd_apply_slab(h, phase: int, nranks: int, rank: int, x_in, x_out, dscale, workspace, stream=None):
    """libfdp slab phase (0 fwd + pack, 1 mid in place, 2 unpack + bwd); see include/fdp.h."""
    _check(lib.fd_apply_slab(h.h, phase, nranks, rank, _dev(x_in, "in"), _dev(x_out, "out"),
                             None if dscale is None else _dev(dscale, "dscale"),
                             _dev(workspace, "workspace"), _stream(stream)))


def kron_mass_apply_slab(h, phase: int, nranks: int, rank: int, x_in, x_out, dscale, workspace,
                         stream=None):
    _check(lib.kron_mass_apply_slab(h.h, phase, nranks, rank, _dev(x_in, "in"), _dev(x_out, "out"),
                                    None if dscale is None else _dev(dscale, "dscale"),
                                    None if workspace is None else _dev(workspace, "workspace"),
                                    _stream(stream)))


def fd_apply_slab_peer(h, phase: int, nranks: int, rank: int, x_in, x_out, peers, dscale, workspace,
                       stream=None):
    """libfdp peer-store slab phase (exchange fused into the epilogue); see include/fdp.h.
    peers: int64 cuda tensor of nranks device addresses (or None in phase 2)."""
    _check(lib.fd_apply_slab_peer(h.h, phase, nranks, rank, _dev(x_in, "in"),
                                  None if x_out is None else _dev(x_out, "out"),
                                  None if peers is None else peers.data_ptr(),
                                  None if dscale is None else _dev(dscale, "dscale"),
                                  _dev(workspace, "workspace"), _stream(stream)))


def kron_mass_apply_slab_peer(h, phase: int, nranks: int, rank: int, x_in, x_out, peers, dscale,
                              workspace, stream=None):
    _check(lib.kron_mass_apply_slab_peer(h.h, phase, nranks, rank, _dev(x_in, "in"),
                                         None if x_out is None else _dev(x_out, "out"),
                                         None if peers is None else peers.data_ptr(),
                                         None if dscale is None else _dev(dscale, "dscale"),
                                         None if workspace is None else _dev(workspace, "workspace"),
                                         _stream(stream)))


class KronMass:
    """kron_mass_setup / kron_mass_apply: P_Q = M_D (x) .. (x) M_1 and its inverse."""

    def __init__(self, Ms, device: int = 0):
        D = len(Ms)
        self.D = D
        self.dims = [int(M.shape[0]) for M in Ms]
        self._M = [_fortran(M) for M in Ms]
        n = (ctypes.c_int32 * D)(*self.dims)
        Mp = (ctypes.c_void_p * D)(*[m.ctypes.data for m in self._M])
        h = ctypes.c_void_p()
        _check(lib.kron_mass_setup(D, n, Mp, device, ctypes.byref(h)))
        self.h = h
        self.N = int(lib.kron_mass_size(h))
        self.device = device

    def apply(self, b, x=None, mode: int = FDP_MASS_INVERSE, dscale=None, batch: int = 1, stream=None):
        import torch
        if x is None:
            x = torch.empty_like(b)
        numel = self.N * batch
        _check(lib.kron_mass_apply(self.h, mode, _dev(b, "b", numel), _dev(x, "x", numel),
                                   None if dscale is None else _dev(dscale, "dscale", self.N),
                                   batch, _stream(stream)))
        return x

    def close(self):
        if getattr(self, "h", None):
            lib.kron_mass_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class BlockPrecond:
    """block_precond_setup / _apply: P_D^{-1} r (or (P_D^G)^{-1} r).

    Owns its FD / KronMass sub-handles (kept alive for the block's lifetime)."""

    def __init__(self, fds, mass, dscale_vel=None, dscale_pres=None):
        D = len(fds)
        self.D = D
        self.fds = list(fds)
        self.mass = mass
        hv = (ctypes.c_void_p * D)(*[f.h.value for f in fds])
        self._dv = None if dscale_vel is None else _host(dscale_vel)
        self._dq = None if dscale_pres is None else _host(dscale_pres)
        h = ctypes.c_void_p()
        _check(lib.block_precond_setup(D, hv, mass.h, None if self._dv is None else _ptr(self._dv),
                                       None if self._dq is None else _ptr(self._dq), ctypes.byref(h)))
        self.h = h
        self.size = int(lib.block_precond_size(h))
        self.sizes = [f.N for f in fds] + [mass.N]
        self.device = mass.device

    def workspace_bytes(self, batch: int = 1) -> int:
        return int(lib.block_precond_workspace_bytes(self.h, batch))

    def workspace(self, batch: int = 1):
        import torch
        return torch.empty(max(1, self.workspace_bytes(batch) // 8), dtype=torch.float64,
                           device=f"cuda:{self.device}")

    def launch_count(self, batch: int = 1) -> int:
        return int(lib.fdp_block_launch_count(self.h, batch))

    def profile(self, enable: bool = True):
        _check(lib.block_precond_profile(self.h, 1 if enable else 0))

    def profile_read(self):
        """[(kind, ms, flops, bytes)] of the last apply (after a stream sync)."""
        cap = 64
        kind = np.zeros(cap, dtype=np.int32)
        ms = np.zeros(cap, dtype=np.float32)
        fl = np.zeros(cap)
        by = np.zeros(cap)
        n = lib.block_precond_profile_read(self.h, cap, _ptr(kind), _ptr(ms), _ptr(fl), _ptr(by))
        if n < 0:
            raise FdpError(5, "profile_read failed (profiling off or events not complete)")
        return [(int(kind[i]), float(ms[i]), float(fl[i]), float(by[i])) for i in range(n)]

    def apply(self, r, s=None, batch: int = 1, workspace=None, stream=None):
        import torch
        if s is None:
            s = torch.empty_like(r)
        if workspace is None:
            workspace = self.workspace(batch)
        numel = self.size * batch
        _check(lib.block_precond_apply(self.h, _dev(r, "r", numel), _dev(s, "s", numel), batch,
                                       _dev(workspace, "workspace", self.workspace_bytes(batch) // 8),
                                       _stream(stream)))
        return s

    def tri(self, variant: str, B, BT):
        """The block-triangular ("T") or constrained ("C") preconditioner built on this block's
        P_V, P_Q and the system's divergence blocks B[k], BT[k] (KronOp, sign included)."""
        return BlockTri(self, variant, B, BT)

    def apply_host(self, r_host: np.ndarray, s_host: np.ndarray, batch: int = 1, stream=None):
        """End-to-end call with host buffers (H2D, apply, D2H, stream sync inside libfdp)."""
        if r_host.dtype != np.float64 or s_host.dtype != np.float64:
            raise TypeError("apply_host: float64 buffers required")
        if not (r_host.flags.c_contiguous and s_host.flags.c_contiguous):
            raise TypeError("apply_host: contiguous buffers required")
        _check(lib.block_precond_apply_host(self.h, ctypes.c_void_p(r_host.ctypes.data),
                                            ctypes.c_void_p(s_host.ctypes.data), batch, _stream(stream)))
        return s_host

    def close(self):
        if getattr(self, "h", None):
            lib.block_precond_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ----------------------------------------------------------------------------------------------
# discretization (product side; built from libfdp's own univariate assembly)
# ----------------------------------------------------------------------------------------------
@dataclass
class Discretization:
    D: int
    disc: str
    p: int
    n_el: int
    Ks: list = field(default_factory=list)     # per component: list of D factors (direction d)
    Ms: list = field(default_factory=list)
    coef: list = field(default_factory=list)
    grev: list = field(default_factory=list)
    Mq: list = field(default_factory=list)
    grev_q: list = field(default_factory=list)

    @property
    def comp_dims(self):
        return [[K.shape[0] for K in Kc] for Kc in self.Ks]

    @property
    def q_dims(self):
        return [M.shape[0] for M in self.Mq]

    @property
    def sizes(self):
        return [int(np.prod(d)) for d in self.comp_dims] + [int(np.prod(self.q_dims))]

    @property
    def n_total(self):
        return int(sum(self.sizes))


def discretization(D: int, disc: str, p: int, n_el: int, rt_own_alpha: int | None = None) -> Discretization:
    """Pencils of P_V,k and P_Q with alpha = p-1, C_pen = 5p.

    TH: velocity degree p+1 interior in every direction, c_d = 1 + [d = k].
    RT component k: degree p+1 / regularity p interior in direction k; degree p full with the
    Nitsche K~ elsewhere."""
    a = p - 1
    out = Discretization(D, disc, p, n_el)
    if disc == "TH":
        K, M = iga_univariate(p + 1, a, n_el, FDP_IGA_INTERIOR)
        g = iga_greville(p + 1, a, n_el, FDP_IGA_INTERIOR)
        for k in range(D):
            out.Ks.append([K] * D)
            out.Ms.append([M] * D)
            out.coef.append([1.0 + (d == k) for d in range(D)])
            out.grev.append([g] * D)
    elif disc == "RT":
        ao = a + 1 if rt_own_alpha is None else rt_own_alpha
        Kn, Mn = iga_univariate(p + 1, ao, n_el, FDP_IGA_INTERIOR)
        Kt, Mt = iga_univariate(p, a, n_el, FDP_IGA_NITSCHE, 5.0 * p)
        gn = iga_greville(p + 1, ao, n_el, FDP_IGA_INTERIOR)
        gt = iga_greville(p, a, n_el)
        for k in range(D):
            out.Ks.append([Kn if d == k else Kt for d in range(D)])
            out.Ms.append([Mn if d == k else Mt for d in range(D)])
            out.coef.append([1.0 + (d == k) for d in range(D)])
            out.grev.append([gn if d == k else gt for d in range(D)])
    else:
        raise ValueError(disc)
    _, Mq = iga_univariate(p, a, n_el)
    out.Mq = [Mq] * D
    out.grev_q = [iga_greville(p, a, n_el)] * D
    return out


def kron_diag(dims, terms, invert: bool = False) -> np.ndarray:
    """libfdp fdp_kron_diag: sum_t c_t prod_d f_td(x_d) sampled on a tensor grid of dof points.
    terms: [(c_t, [values of f_td at direction d's points, or None for 1])]."""
    D = len(dims)
    n = (ctypes.c_int32 * D)(*dims)
    keep = []
    fp = (ctypes.c_void_p * (D * len(terms)))()
    for t, (_, fs) in enumerate(terms):
        for d in range(D):
            v = None if fs is None else fs[d]
            if v is not None:
                v = np.ascontiguousarray(v, dtype=np.float64)
                assert v.shape == (dims[d],)
                keep.append(v)
                fp[t * D + d] = v.ctypes.data
    c = np.array([ct for ct, _ in terms], dtype=np.float64)
    out = np.empty(int(np.prod(dims)), dtype=np.float64)
    _check(lib.fdp_kron_diag(D, n, len(terms), fp, _ptr(c), int(invert), _ptr(out)))
    return out


def nu_scalings(d: Discretization, terms):
    """Config 3 (C-6): D_V = nu at the velocity dofs' Greville points, D_Q = 1/nu at the
    pressure dofs', for nu given as separable terms [(c_t, [w_t1, .., w_tD])] (w = None: 1),
    e.g. synth.viscosity_separable(D); the tensor-grid sampling runs in libfdp (fdp_kron_diag)."""
    if callable(terms):
        raise TypeError("nu_scalings takes nu as separable terms (synth.viscosity_separable)")

    def sampled(grevs):
        return [(c, None if ws is None else [w(g) for w, g in zip(ws, grevs)]) for c, ws in terms]

    dv = np.concatenate([kron_diag([len(g) for g in gr], sampled(gr)) for gr in d.grev])
    dq = kron_diag([len(g) for g in d.grev_q], sampled(d.grev_q), invert=True)
    return dv, dq


def build_block(d: Discretization, device: int = 0, dscale_vel=None, dscale_pres=None) -> BlockPrecond:
    fds = [FD(d.Ks[k], d.Ms[k], d.coef[k], device=device) for k in range(d.D)]
    mass = KronMass(d.Mq, device=device)
    return BlockPrecond(fds, mass, dscale_vel, dscale_pres)


FDP_PREC_TRIANGULAR = 1
FDP_PREC_CONSTRAINED = 2


class BlockTri:
    """block_tri_apply: s = P_T^{-1} r or P_C^{-1} r, batch 1."""

    def __init__(self, block: "BlockPrecond", variant: str, B, BT):
        self.block = block
        self.variant = {"T": FDP_PREC_TRIANGULAR, "C": FDP_PREC_CONSTRAINED}[variant]
        self.B, self.BT = list(B), list(BT)
        self._hB = KronOp._handles(self.B)
        self._hBT = KronOp._handles(self.BT)
        self.size = block.size
        nb = int(lib.block_tri_workspace_bytes(block.h, self.variant, self._hB, self._hBT))
        if nb == 0:
            raise FdpError(1, "block_tri_workspace_bytes: " + lib.fdp_last_error().decode())
        self._ws_bytes = nb

    def workspace(self):
        import torch
        return torch.empty(self._ws_bytes // 8 + 1, dtype=torch.float64,
                           device=f"cuda:{self.block.device}")

    def apply(self, r, s, workspace, stream=None):
        _check(lib.block_tri_apply(self.block.h, self.variant, self._hB, self._hBT,
                                   _dev(r, "r", self.size), _dev(s, "s", self.size),
                                   _dev(workspace, "workspace", self._ws_bytes // 8), _stream(stream)))
        return s
