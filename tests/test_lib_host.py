"""CPU-side checks of libfdp: the shared library loads, exports every symbol include/fdp.h
declares, and its host numerics (univariate assembly, Greville points, generalized eigensolver)
agree with the oracle. No compute kernels run here."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1712_00403_b200 as fdp
from oracle import fd as ofd
from oracle import splines, univariate

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "fdp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(\w+)\s*\(", src, flags=re.M)
    return sorted(set(n for n in names if n not in ("if", "defined")))


def test_header_symbols_exported():
    out = subprocess.run(["nm", "-D", "--defined-only", fdp.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(l.split()[-1] for l in out.splitlines() if " T " in l)
    declared = _declared()
    assert len(declared) >= 20
    missing = [n for n in declared if n not in exported]
    assert not missing, missing


def test_status_strings_and_version():
    assert fdp.lib.fdp_status_string(0) == b"FDP_OK"
    assert fdp.lib.fdp_status_string(4) == b"FDP_ERR_SINGULAR"
    assert b"sm_100a" in fdp.lib.fdp_version()


@pytest.mark.parametrize("deg,alpha,n_el,flags", [(3, 1, 16, 1), (4, 2, 32, 1), (5, 4, 64, 1),
                                                   (4, 3, 64, 0), (6, 4, 20, 1), (2, 0, 5, 0), (1, 0, 3, 1)])
def test_iga_univariate_matches_oracle(deg, alpha, n_el, flags):
    K, M = fdp.iga_univariate(deg, alpha, n_el, flags)
    Ko, Mo = univariate.stiffness_mass(deg, alpha, n_el)
    if flags & 1:
        Ko, Mo = univariate.interior(Ko), univariate.interior(Mo)
    assert K.shape == Ko.shape
    assert np.max(np.abs(K - Ko)) <= 1e-13 * np.max(np.abs(Ko))
    assert np.max(np.abs(M - Mo)) <= 1e-13 * np.max(np.abs(Mo))


@pytest.mark.parametrize("p,n_el", [(1, 1), (2, 4), (4, 64), (4, 512)])
def test_iga_nitsche_matches_oracle(p, n_el):
    K, M = fdp.iga_univariate(p, p - 1, n_el, fdp.FDP_IGA_NITSCHE, 5.0 * p)
    Ko = univariate.nitsche_stiffness(p, p - 1, n_el, univariate.c_pen(p))
    assert np.max(np.abs(K - Ko)) <= 1e-13 * np.max(np.abs(Ko))


def test_greville_matches_oracle():
    for deg, a, n, fl in [(4, 2, 8, 1), (4, 3, 8, 0), (5, 4, 6, 1)]:
        g = fdp.iga_greville(deg, a, n, fl)
        go = splines.greville(splines.open_uniform_knots(deg, a, n), deg)
        if fl:
            go = go[1:-1]
        assert np.allclose(g, go, rtol=0, atol=1e-15)


@pytest.mark.parametrize("pencil", ["th65", "rt_t68", "rt_n67", "q35"])
def test_gen_eig_matches_oracle(pencil):
    K, M = {"th65": lambda: univariate.th_velocity_pencil(3, 32),
            "rt_t68": lambda: univariate.rt_tangential_pencil(4, 64),
            "rt_n67": lambda: univariate.rt_normal_pencil(4, 64),
            "q35": lambda: univariate.stiffness_mass(3, 2, 32)}[pencil]()
    lam, U = fdp.gen_eig(K, M)
    lo, _ = ofd.gen_eig(K, M)
    assert np.max(np.abs(lam - lo) / np.abs(lo).max()) < 1e-13
    assert np.max(np.abs(U.T @ M @ U - np.eye(len(lam)))) < 1e-12
    assert np.max(np.abs(K @ U - M @ U * lam)) < 1e-11 * np.abs(lo).max()


def test_gen_eig_rejects_non_spd():
    with pytest.raises(fdp.FdpError) as e:
        fdp.gen_eig(np.eye(3), -np.eye(3))
    assert e.value.status == 3  # FDP_ERR_NOT_SPD


def test_setup_argument_errors_without_gpu():
    h = ctypes.c_void_p()
    n = (ctypes.c_int32 * 4)(2, 2, 2, 2)
    assert fdp.lib.fd_setup(4, n, None, None, None, 0, 0, ctypes.byref(h)) == 8   # UNSUPPORTED
    assert fdp.lib.fd_setup(3, None, None, None, None, 0, 0, ctypes.byref(h)) == 1  # INVALID_ARG
    n0 = (ctypes.c_int32 * 3)(0, 2, 2)
    K = np.eye(2)
    Kp = (ctypes.c_void_p * 3)(*[K.ctypes.data] * 3)
    c = (ctypes.c_double * 3)(1, 1, 1)
    assert fdp.lib.fd_setup(3, n0, Kp, Kp, c, 0, 0, ctypes.byref(h)) == 2         # SHAPE
    assert fdp.lib.kron_mass_setup(1, n0, Kp, 0, ctypes.byref(h)) == 8
    assert fdp.lib.iga_univariate(0, 0, 1, 0, 0.0, 0, None, None, ctypes.byref(ctypes.c_int32())) == 2


def test_discretization_matches_oracle_sizes():
    import synth
    from oracle import spaces
    for cid in (1, 2, 3):
        w = synth.CONFIGS[cid]
        g = fdp.discretization(w.dim, w.disc, w.p, w.n_el)
        o = spaces.build(w.dim, w.disc, w.p, w.n_el)
        assert g.comp_dims == [c.dims for c in o.comps]
        assert g.n_total == o.n_total
        assert g.coef == [c.coef for c in o.comps]


@pytest.mark.parametrize("case", [
    ((3, 1, 1), (3, 1, 1), 0, 1), ((2, 1, 0), (3, 1, 1), 0, 1), ((2, 1, 0), (3, 1, 1), 0, 0),
    ((4, 3, 1), (3, 2, 0), 1, 0), ((5, 4, 1), (5, 4, 1), 1, 1)])
def test_iga_mixed_matches_oracle(case):
    from oracle import stokes as ost
    (dt, at, ft), (dr, ar, fr), dtest, dtrial = case
    n_el = 5
    q = max(dt, dr) + 3
    A = fdp.iga_mixed((dt, at, ft), (dr, ar, fr), n_el, dtest, dtrial, q)
    Ao = ost._mixed(ost._space(dt, at, n_el, bool(ft & 1)), ost._space(dr, ar, n_el, bool(fr & 1)),
                    n_el, q, bool(dtest), bool(dtrial))
    assert A.shape == Ao.shape
    assert np.max(np.abs(A - Ao)) <= 1e-13 * np.max(np.abs(Ao))


def test_iga_mixed_weighted_and_quadrature():
    from oracle import stokes as ost
    n_el, q = 6, 7
    x, w = fdp.iga_quadrature(n_el, q)
    assert abs(w.sum() - 1.0) < 1e-14 and np.all((x > 0) & (x < 1))
    wt = np.sin(2 * np.pi * x)
    A = fdp.iga_mixed((3, 2, 1), (3, 2, 1), n_el, 1, 1, q, wt)
    Ao = ost._mixed(ost._space(3, 2, n_el, True), ost._space(3, 2, n_el, True), n_el, q, True, True,
                    weight=lambda t: np.sin(2 * np.pi * t))
    assert np.max(np.abs(A - Ao)) <= 1e-13 * np.max(np.abs(Ao))


def test_geometry_coeffs_and_separable_fit_match_oracle():
    """NEXT-3 host helpers (iga_geometry_coeffs, iga_separable_fit) vs oracle/geometry.py."""
    from oracle import geometry as og
    x, _ = og.quadrature_grid(3, 5)
    for k in range(3):
        c_o = og.sample_diagonal(og.annulus(), k, x)
        c_l = fdp.iga_geometry_coeffs(fdp.FDP_GEOM_ANNULUS, 3, k, x)
        for d in range(3):
            ref = np.reshape(c_o[d], -1, order="F")
            assert np.max(np.abs(c_l[d] - ref) / ref) < 1e-14
        t_o, m_o, _ = og.separable_fit(c_o)
        t_l, m_l, _ = fdp.iga_separable_fit(c_l, [x.size] * 3)
        for a, b in zip(t_o + m_o, t_l + m_l):
            assert np.max(np.abs(a - b) / b) < 1e-12
        ci = fdp.iga_geometry_coeffs(fdp.FDP_GEOM_IDENTITY, 3, k, x)
        for d in range(3):
            assert np.all(ci[d] == (2.0 if d == k else 1.0))


def test_separable_fit_rejects_nonpositive():
    c = [np.ones(8), np.ones(8)]
    c[1][3] = 0.0
    with pytest.raises(fdp.FdpError):
        fdp.iga_separable_fit(c, [2, 4])


def test_header_is_plain_c99(tmp_path):
    """include/fdp.h is a C99 header: it compiles as C with -pedantic, and a C
    program can call the host-only entry points through it."""
    src = tmp_path / "t.c"
    src.write_text('#include "fdp.h"\n#include <stdio.h>\nint main(void) {\n'
                   '  int32_t n = 0;\n  fdp_status s = iga_univariate(2, 1, 4, 0, 0.0, 0, NULL, NULL, &n);\n'
                   '  printf("%d %d %s\\n", (int)s, (int)n, fdp_version());\n  return s != FDP_OK;\n}\n')
    inc = os.path.join(ROOT, "include")
    libdir = os.path.dirname(fdp.LIB_PATH)
    exe = tmp_path / "t"
    r = subprocess.run(["gcc", "-std=c99", "-pedantic", "-Wall", "-Werror", "-I", inc, str(src), "-o", str(exe),
                        "-L", libdir, "-lfdp", f"-Wl,-rpath,{libdir}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert out.stdout.split()[1] == "6"   # m = n_el (p - alpha) + alpha + 1 = 4 + 1 + 1


def test_setup_validation_paths_without_gpu():
    """Argument checks that run before any device work: extents above the 2048 limit, non-positive
    coefficients, non-symmetric pencils, block / Kronecker / communicator misuse, slab ranks."""
    h = ctypes.c_void_p()
    K = np.eye(3)
    Kp = (ctypes.c_void_p * 3)(*[K.ctypes.data] * 3)
    c = (ctypes.c_double * 3)(1, 1, 1)
    big = (ctypes.c_int32 * 3)(2049, 3, 3)
    assert fdp.lib.fd_setup(3, big, Kp, Kp, c, 0, 0, ctypes.byref(h)) == 2           # SHAPE
    n3 = (ctypes.c_int32 * 3)(3, 3, 3)
    c0 = (ctypes.c_double * 3)(1, 0, 1)
    assert fdp.lib.fd_setup(3, n3, Kp, Kp, c0, 0, 0, ctypes.byref(h)) == 1           # coef <= 0
    A = np.array([[2.0, 1.0, 0.0], [0.0, 2.0, 0.0], [0.0, 0.0, 2.0]], order="F")
    Ap = (ctypes.c_void_p * 3)(*[A.ctypes.data] * 3)
    assert fdp.lib.fd_setup(3, n3, Ap, Kp, c, 0, 0, ctypes.byref(h)) == 3            # NOT_SPD (asym.)
    assert fdp.lib.fd_setup(3, n3, Kp, Kp, c, 0, -1, ctypes.byref(h)) == 2           # max_batch < 0
    assert fdp.lib.block_precond_setup(3, None, None, None, None, ctypes.byref(h)) == 1
    assert fdp.lib.block_precond_setup(4, None, None, None, None, ctypes.byref(h)) == 8
    assert fdp.lib.kron_op_setup(2, 0, n3, n3, Kp, c, 0, ctypes.byref(h)) == 1        # no terms
    assert fdp.lib.kron_op_setup(2, 1, big, n3, Kp, c, 0, ctypes.byref(h)) == 2       # extent
    assert fdp.lib.fdp_comm_create(None, 2, 0, ctypes.byref(h), ctypes.create_string_buffer(8)) == 1
    lo, ln = ctypes.c_int64(), ctypes.c_int64()
    assert fdp.lib.fdp_slab_range(10, 3, 3, ctypes.byref(lo), ctypes.byref(ln)) == 1  # rank >= G
    assert fdp.lib.fdp_slab_range(10, 3, 2, ctypes.byref(lo), ctypes.byref(ln)) == 0
    assert (lo.value, ln.value) == (7, 3)
    assert fdp.lib.fd_destroy(None) == 0 and fdp.lib.block_precond_destroy(None) == 0
    assert fdp.lib.fdp_comm_destroy(None) == 0 and fdp.lib.kron_op_destroy(None) == 0
    assert fdp.lib.fdp_last_error()  # a message was recorded


def test_mass_diag_factor_matches_oracle():
    """iga_mass_diag_factor: w_g b_i(x_g)^2 at the element Gauss points; its row sums are the
    diagonal of the unweighted mass matrix."""
    from oracle import splines
    for deg, alpha, n_el, q in [(2, 1, 4, 3), (4, 3, 6, 7), (3, 1, 5, 5)]:
        F = fdp.iga_mass_diag_factor((deg, alpha, 0), n_el, q)
        xi = splines.open_uniform_knots(deg, alpha, n_el)
        x, w = splines.element_quadrature(np.linspace(0, 1, n_el + 1), q)
        ref = (w[:, None] * splines.basis(xi, deg, x) ** 2).T
        assert np.max(np.abs(F - ref)) < 1e-14
        _, M = univariate.stiffness_mass(deg, alpha, n_el)
        assert np.max(np.abs(F.sum(axis=1) - np.diag(M))) < 1e-14


def test_library_nu_scalings_pinned_axis_asymmetric():
    """libfdp's D_V / D_Q sampling (fdp_kron_diag over iga_greville points, a different code path
    from the oracle's meshgrid) against the same hand-evaluated RT p = 2, n_el = 2 values as
    tests/test_oracle_mass_block.py (C-6)."""
    g_own, g_tan = [1 / 6, 1 / 2, 5 / 6], [0.0, 1 / 4, 3 / 4, 1.0]
    nu = lambda x, y, z: 1.0 + x + 10.0 * y + 100.0 * z
    ident = lambda x: np.asarray(x, dtype=float)
    terms = [(1.0, None), (1.0, [ident, None, None]), (10.0, [None, ident, None]),
             (100.0, [None, None, ident])]
    terms = [(c, None if ws is None else [w if w is not None else (lambda x: np.ones(len(x)))
                                          for w in ws]) for c, ws in terms]
    gd = fdp.discretization(3, "RT", 2, 2)
    dv, dq = fdp.nu_scalings(gd, terms)
    off = 0
    for k in range(3):
        g = [g_own if d == k else g_tan for d in range(3)]
        exp = [nu(g[0][i1], g[1][i2], g[2][i3])
               for i3 in range(len(g[2])) for i2 in range(len(g[1])) for i1 in range(len(g[0]))]
        np.testing.assert_allclose(dv[off:off + len(exp)], exp, rtol=1e-14)
        off += len(exp)
    expq = [1 / nu(g_tan[i1], g_tan[i2], g_tan[i3]) for i3 in range(4) for i2 in range(4) for i1 in range(4)]
    np.testing.assert_allclose(dq, expq, rtol=1e-14)
    with pytest.raises(TypeError):
        fdp.nu_scalings(gd, nu)


def test_library_nu_scalings_config3_matches_oracle():
    """Config-3-shaped sampling (RT p = 4, small n_el) of synth's nu: library (separable terms,
    fdp_kron_diag) vs oracle (nu evaluated on the meshgrid)."""
    import synth
    from oracle import spaces
    gd = fdp.discretization(3, "RT", 4, 5)
    od = spaces.build(3, "RT", 4, 5)
    dv, dq = fdp.nu_scalings(gd, synth.viscosity_separable(3))
    odv, odq = spaces.nu_scalings(od, synth.viscosity)
    np.testing.assert_allclose(dv, odv, rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(dq, odq, rtol=1e-14)
