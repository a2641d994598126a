"""Memory-safety evidence without compute-sanitizer (closed on this GPU pool: runs under it left
GPUs needing a reset): every buffer an apply touches lives inside a larger allocation whose
margins hold a NaN sentinel bit pattern, the workspace and the output are poisoned with the same
NaN, and the inputs sit at aligned and at odd (8-byte-only) offsets. After the apply
  * the margins must be bit-identical (no out-of-bounds write, before or after any buffer),
  * every output element must be finite and equal the oracle's (every element written; no read
    of a workspace element the apply did not write first -- a NaN read would propagate through
    the contractions: NaN x 0 = NaN),
  * the input must be unchanged (no stray write into it).
Covers the plane / small paths (configs 1-3, P^G), K1t with its row-padding pass and the K1f
fallback (random persymmetric pencils of config 4/5 extents), the banded pressure solves, and
config 4 at full size in the bench launch (batch 8)."""
import numpy as np
import pytest
import torch

import paper_1712_00403_b200 as fdp
import synth
from oracle import fd as ofd
from oracle import mass as omass
from oracle import precond as oprec
from oracle import spaces as ospaces

pytestmark = pytest.mark.gpu

GUARD = 4096                      # sentinel doubles on each side of every buffer
SENT = 0x7FF8DEADBEEF1234         # a quiet NaN with a recognisable payload (a positive int64)
TOL = 1e-9


def _guarded(n, fill=None, odd=False):
    """(whole allocation, view of n doubles) with sentinel margins; odd: the view starts at an
    8-byte but not 16-byte aligned address."""
    off = GUARD + (1 if odd else 0)
    buf = torch.empty(n + 2 * GUARD + 2, dtype=torch.float64, device="cuda")
    buf.view(torch.int64).fill_(SENT)
    view = buf[off:off + n]
    if fill is not None:
        view.copy_(torch.as_tensor(np.ascontiguousarray(fill).reshape(-1), dtype=torch.float64))
    return buf, view, off


def _margins_intact(buf, off, n):
    raw = buf.view(torch.int64)
    return bool((raw[:off] == SENT).all().item() and (raw[off + n:] == SENT).all().item())


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def relmax(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


@pytest.mark.parametrize("cid,batch,scaled,odd", [(1, 1, False, False), (1, 2, False, True),
                                                  (2, 1, False, False), (2, 2, False, True),
                                                  (3, 1, True, False), (3, 1, True, True)])
def test_block_apply_guards_and_poisoned_workspace(cid, batch, scaled, odd):
    w = synth.CONFIGS[cid]
    od = ospaces.build(w.dim, w.disc, w.p, w.n_el)
    gd = fdp.discretization(w.dim, w.disc, w.p, w.n_el)
    dv = dq = None
    if scaled:
        dv, dq = ospaces.nu_scalings(od, synth.viscosity)
    P = fdp.build_block(gd, dscale_vel=dv, dscale_pres=dq)
    n = od.n_total * batch
    r = np.random.default_rng(cid + 10 * batch).standard_normal((batch, od.n_total))
    rb, rv, ro = _guarded(n, r, odd)
    sb, sv, so = _guarded(n, None, odd)
    sv.view(torch.int64).fill_(SENT)
    wn = P.workspace_bytes(batch) // 8 + 1
    wb, wv, wo = _guarded(wn, None)
    wv.view(torch.int64).fill_(SENT)
    P.apply(rv, sv, batch=batch, workspace=wv)
    torch.cuda.synchronize()
    for buf, off, m in ((rb, ro, n), (sb, so, n), (wb, wo, wn)):
        assert _margins_intact(buf, off, m)
    assert np.array_equal(rv.cpu().numpy(), r.reshape(-1))
    s = sv.cpu().numpy().reshape(batch, -1)
    assert np.all(np.isfinite(s))
    ref = oprec.BlockPrecond(od, dv, dq) if scaled else oprec.BlockPrecond(od)
    for i in range(batch):
        x = ref.apply(r[i])
        assert rel(s[i], x) < TOL and relmax(s[i], x) < TOL


def _persym_spd(n, rng, shift):
    a = rng.standard_normal((n, n))
    a = a @ a.T + shift * n * np.eye(n)
    return 0.5 * (a + a[::-1, ::-1])


@pytest.mark.parametrize("dims,batch,odd,env", [
    ((259, 130, 97), 2, True, {}),            # K1t after the row-padding pass (odd rows, odd base)
    ((260, 131, 99), 1, False, {}),           # K1t reading the C-ABI input in place
    ((9, 7, 516), 2, True, {}),               # the Lambda pass (1/Lambda table) at config 5's extent
    ((130, 300, 97), 1, False, {"FDP_NO_TMA": "1"}),  # the cp.async K1f fallback
])
def test_fd_guards_and_poisoned_workspace(dims, batch, odd, env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(sum(dims) + batch)
    Ks = [_persym_spd(n, rng, 1.0) for n in dims]
    Ms = [_persym_spd(n, rng, 2.0) for n in dims]
    coef = (2.0, 1.0, 1.0)
    N = int(np.prod(dims))
    F = fdp.FD(Ks, Ms, coef)
    b = rng.standard_normal((batch, N))
    dsc = rng.uniform(0.5, 1.5, N)
    bb, bv, bo = _guarded(N * batch, b, odd)
    xb, xv, xo = _guarded(N * batch, None, odd)
    db, dvw, do = _guarded(N, 1.0 / np.sqrt(dsc), odd)
    wn = F.workspace_bytes(batch) // 8 + 1
    wb, wv, wo = _guarded(wn, None)
    wv.view(torch.int64).fill_(SENT)
    xv.view(torch.int64).fill_(SENT)
    F.apply(bv, xv, dscale=dvw, batch=batch, workspace=wv)
    torch.cuda.synchronize()
    for buf, off, m in ((bb, bo, N * batch), (xb, xo, N * batch), (db, do, N), (wb, wo, wn)):
        assert _margins_intact(buf, off, m)
    x = xv.cpu().numpy().reshape(batch, N)
    assert np.all(np.isfinite(x))
    ref = ofd.FDSolver(Ks, Ms, coef)
    for i in range(batch):
        xr = ofd.scaled_apply(ref, b[i], dsc)
        assert rel(x[i], xr) < TOL and relmax(x[i], xr) < TOL


def test_banded_mass_guards():
    """The banded per-mode pressure solves (K3) on a config-3-sized pressure block, odd base."""
    od = ospaces.build(3, "RT", 4, 16)
    Mq = od.Mq
    M = fdp.KronMass(Mq)
    n = int(np.prod([m.shape[0] for m in Mq]))
    b = np.random.default_rng(7).standard_normal(n)
    bb, bv, bo = _guarded(n, b, True)
    xb, xv, xo = _guarded(n, None, True)
    xv.view(torch.int64).fill_(SENT)
    M.apply(bv, xv)
    torch.cuda.synchronize()
    assert _margins_intact(bb, bo, n) and _margins_intact(xb, xo, n)
    x = xv.cpu().numpy()
    ref = omass.KronMass(Mq).inverse(b)
    assert np.all(np.isfinite(x))
    assert rel(x, ref) < TOL and relmax(x, ref) < TOL


@pytest.mark.parametrize("pn,batch,scaled", [
    (((3, 25), (2, 30), (1, 19)), 2, False),  # n = 28, 32, 20: ragged 12-fiber tiles in every mode, batch
    (((4, 124), (4, 124)), 1, True),          # 2D, n = 128 x 128: ragged tiles (128 = 10 x 12 + 8), P^G scaling
])
def test_k3u_tile_kernel_guards(pn, batch, scaled):
    """K3u (the persistent tile kernel of the banded pressure solve: bulk copies and tensor-map
    boxes in and out of shared memory) on 16-byte-aligned guarded buffers: margins intact, every
    output finite and equal to the oracle's."""
    from oracle import univariate
    Mq = [univariate.pressure_mass(p, ne) for p, ne in pn]
    M = fdp.KronMass(Mq)
    n = int(np.prod([m.shape[0] for m in Mq]))
    rng = np.random.default_rng(11)
    b = rng.standard_normal((batch, n))
    dq = rng.uniform(0.5, 2.0, n)
    bb, bv, bo = _guarded(n * batch, b, False)
    xb, xv, xo = _guarded(n * batch, None, False)
    db, dvw, do = _guarded(n, 1.0 / np.sqrt(dq), False)
    xv.view(torch.int64).fill_(SENT)
    M.apply(bv, xv, dscale=dvw if scaled else None, batch=batch)
    torch.cuda.synchronize()
    assert _margins_intact(bb, bo, n * batch) and _margins_intact(xb, xo, n * batch) and _margins_intact(db, do, n)
    x = xv.cpu().numpy().reshape(batch, n)
    assert np.all(np.isfinite(x))
    km = omass.KronMass(Mq)
    for i in range(batch):
        ref = km.scaled_inverse(b[i], dq) if scaled else km.inverse(b[i])
        assert rel(x[i], ref) < TOL and relmax(x[i], ref) < TOL


@pytest.mark.slow
def test_config4_bench_launch_guards():
    """Config 4 at full size in the bench launch (batch 8, 436 M doubles per vector): guards and a
    NaN-poisoned workspace; every output finite, items 0 and 7 against the oracle."""
    w = synth.CONFIGS[4]
    od = ospaces.build(w.dim, w.disc, w.p, w.n_el)
    gd = fdp.discretization(w.dim, w.disc, w.p, w.n_el)
    P = fdp.build_block(gd)
    r = synth.rhs(w.seed, od.n_total, w.batch)
    n = r.size
    rb, rv, ro = _guarded(n, r)
    sb, sv, so = _guarded(n, None)
    sv.view(torch.int64).fill_(SENT)
    wn = P.workspace_bytes(w.batch) // 8 + 1
    wb, wv, wo = _guarded(wn, None)
    wv.view(torch.int64).fill_(SENT)
    P.apply(rv, sv, batch=w.batch, workspace=wv)
    torch.cuda.synchronize()
    for buf, off, m in ((rb, ro, n), (sb, so, n), (wb, wo, wn)):
        assert _margins_intact(buf, off, m)
    s = sv.view(w.batch, -1)
    assert bool(torch.isfinite(s).all())
    del wb, wv
    ref = oprec.BlockPrecond(od)
    for i in (0, 7):
        x = ref.apply(r[i])
        si = s[i].cpu().numpy()
        assert rel(si, x) < TOL and relmax(si, x) < TOL
