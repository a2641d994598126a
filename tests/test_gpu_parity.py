"""GPU parity: libfdp (through the C ABI via the thin binding) vs the CPU oracle, element by
element on the same seeded inputs. Tolerance: relative L2 <= 1e-9 (BASELINE.json north_star);
expected ~1e-14 (two different eigensolvers, FP64 throughout)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1712_00403_b200 as fdp  # noqa: E402
import synth  # noqa: E402
from oracle import fd as ofd  # noqa: E402
from oracle import mass as omass  # noqa: E402
from oracle import precond as oprec  # noqa: E402
from oracle import spaces as ospaces  # noqa: E402

pytestmark = pytest.mark.gpu
TOL = 1e-9


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _rand_spd(n, rng, shift):
    A = rng.standard_normal((n, n))
    return A @ A.T + shift * n * np.eye(n)


@pytest.mark.parametrize("dims,coef,batch", [
    ((37, 70, 19), (2.0, 1.0, 1.0), 3),      # ragged in every mode, several tiles
    ((5, 33, 100), (1.0, 2.0, 1.0), 2),
    ((133, 9, 17), (1.0, 1.0, 2.0), 1),
    ((150, 67), (2.0, 1.0), 4),             # 2D, two column tiles in mode 1
    ((1, 7, 3), (1.0, 1.0, 1.0), 2),        # degenerate extent 1
    ((96, 96, 2), (0.5, 1.5, 3.0), 1),
    ((2048, 3, 2), (1.0, 2.0, 1.0), 1),     # largest extent fd_setup accepts (22 column tiles)
    ((2, 2048), (1.0, 3.0), 2),
])
def test_fd_apply_random_pencils(dims, coef, batch):
    rng = np.random.default_rng(sum(dims) + batch)
    Ks = [_rand_spd(n, rng, 1.0) for n in dims]
    Ms = [_rand_spd(n, rng, 2.0) for n in dims]
    N = int(np.prod(dims))
    b = rng.standard_normal((batch, N))
    S = fdp.FD(Ks, Ms, coef)
    x = S.apply(dev(b), batch=batch).cpu().numpy()
    ref = ofd.FDSolver(Ks, Ms, coef)
    for i in range(batch):
        assert rel(x[i], ref.apply(b[i])) < TOL


def _rand_persym_spd(n, rng, shift):
    A = _rand_spd(n, rng, shift)
    return 0.5 * (A + A[::-1, ::-1])  # J A J = A: the even-odd folded path takes it


@pytest.mark.parametrize("dims,coef,batch,dscale", [
    ((37, 70, 19), (2.0, 1.0, 1.0), 2, False),   # all folded, fused middle pass, odd/even extents
    ((8, 9, 96), (1.0, 2.0, 1.0), 1, True),      # smallest / largest folded extents, P^G scaling
    ((150, 67, 40), (1.0, 1.0, 2.0), 1, False),  # mode 1 dense (> 96): Lambda on a folded forward
    ((65, 65, 65), (2.0, 1.0, 1.0), 1, True),    # config 2's velocity extent
    ((33, 64), (1.0, 2.0), 3, False),            # 2D
    ((7, 12, 20), (1.0, 1.0, 1.0), 1, False),    # 7 < 8 stays dense next to folded modes
    ((259, 20, 9), (2.0, 1.0, 1.0), 2, True),    # K1 folded mode 1 (KMAJ), odd n, P^G scaling
    ((12, 258, 97), (1.0, 2.0, 1.0), 1, False),  # K1 folded modes 2 and 3, Lambda on the K1 fold
    ((300, 2), (1.0, 3.0), 2, False),            # 2D, K1 folded even extent
    ((40, 66, 71), (1.0, 1.0, 2.0), 4, True),    # plane path (160 planes), n2 != n3, batch 4
    ((75, 57, 64), (2.0, 1.0, 1.0), 2, False),   # plane path, leftover rows in both plane steps
    ((40, 66, 71), (1.0, 1.0, 2.0), 1, False),   # 40 planes < one per SM: the five passes
    ((40, 45), (2.0, 1.0), 3, True),             # 2D one-launch plane path, P^G, batch 3
    ((65, 66), (1.0, 2.0), 1, False),            # 2D one-launch plane path, odd / even
])
def test_fd_apply_folded_persymmetric(dims, coef, batch, dscale):
    """Even-odd folded transforms on random persymmetric SPD pencils: the folded
    apply against the oracle's dense FD (Algorithm 1) and against the library's own dense path
    (FDP_NO_FOLD=1)."""
    import os
    rng = np.random.default_rng(sum(dims) + 7 * batch)
    Ks = [_rand_persym_spd(n, rng, 1.0) for n in dims]
    Ms = [_rand_persym_spd(n, rng, 2.0) for n in dims]
    N = int(np.prod(dims))
    b = rng.standard_normal((batch, N))
    dsc = rng.uniform(0.5, 1.5, N) if dscale else None
    S = fdp.FD(Ks, Ms, coef)
    kw = {"dscale": dev(1.0 / np.sqrt(dsc))} if dscale else {}
    x = S.apply(dev(b), batch=batch, **kw).cpu().numpy()
    os.environ["FDP_NO_FOLD"] = "1"
    try:
        x_dense = fdp.FD(Ks, Ms, coef).apply(dev(b), batch=batch, **kw).cpu().numpy()
    finally:
        del os.environ["FDP_NO_FOLD"]
    ref = ofd.FDSolver(Ks, Ms, coef)
    for i in range(batch):
        r = ofd.scaled_apply(ref, b[i], dsc) if dscale else ref.apply(b[i])
        assert rel(x[i], r) < TOL
        assert rel(x[i], x_dense[i]) < 1e-12


def test_fd_apply_dscale_and_inplace():
    d = ospaces.build(3, "RT", 2, 6)
    c = d.comps[1]
    rng = np.random.default_rng(5)
    N = c.size
    b = rng.standard_normal(N)
    dsc = rng.uniform(0.5, 1.5, N)
    S = fdp.FD(c.Ks, c.Ms, c.coef)
    bt = dev(b)
    S.apply(bt, bt, dscale=dev(1.0 / np.sqrt(dsc)))  # in place
    ref = ofd.scaled_apply(ofd.FDSolver(c.Ks, c.Ms, c.coef), b, dsc)
    assert rel(bt.cpu().numpy(), ref) < TOL


def test_kron_mass_inverse_and_forward():
    rng = np.random.default_rng(8)
    from oracle import univariate
    Ms = [univariate.pressure_mass(3, 5), univariate.pressure_mass(3, 7), univariate.pressure_mass(3, 4)]
    km = omass.KronMass(Ms)
    N = int(np.prod(km.dims))
    b = rng.standard_normal((2, N))
    K = fdp.KronMass(Ms)
    x = K.apply(dev(b), batch=2).cpu().numpy()
    y = K.apply(dev(b), mode=fdp.FDP_MASS_FORWARD, batch=2).cpu().numpy()
    dq = rng.uniform(0.5, 2.0, N)
    z = K.apply(dev(b), dscale=dev(1 / np.sqrt(dq)), batch=2).cpu().numpy()
    for i in range(2):
        assert rel(x[i], km.inverse(b[i])) < TOL
        assert rel(y[i], km.forward(b[i])) < 1e-13
        assert rel(z[i], km.scaled_inverse(b[i], dq)) < TOL


def _both(cfg_id):
    w = synth.CONFIGS[cfg_id]
    od = ospaces.build(w.dim, w.disc, w.p, w.n_el)
    gd = fdp.discretization(w.dim, w.disc, w.p, w.n_el)
    return w, od, gd


@pytest.mark.parametrize("cfg_id", [1, 2, 3])
def test_block_precond_configs(cfg_id):
    w, od, gd = _both(cfg_id)
    assert gd.comp_dims == [c.dims for c in od.comps] and gd.q_dims == od.q_dims
    r = synth.rhs(w.seed, od.n_total, w.batch)
    dv = dq = None
    if w.variable_nu:
        dv, dq = ospaces.nu_scalings(od, synth.viscosity)
        gdv, gdq = fdp.nu_scalings(gd, synth.viscosity_separable(gd.D))
        assert np.max(np.abs(gdv - dv)) < 1e-14 and np.max(np.abs(gdq - dq)) < 1e-14
    P = fdp.build_block(gd, dscale_vel=dv, dscale_pres=dq)
    s = P.apply(dev(r), batch=w.batch).cpu().numpy()
    ref = oprec.BlockPrecond(od, dv, dq).apply(r)
    o = od.offsets()
    for i in range(w.batch):
        for k in range(len(o) - 1):
            assert rel(s[i, o[k]:o[k + 1]], ref[i, o[k]:o[k + 1]]) < TOL, (cfg_id, k)
            assert relmax(s[i, o[k]:o[k + 1]], ref[i, o[k]:o[k + 1]]) < TOL, (cfg_id, k)


def test_block_precond_plain_vs_scaled_config3():
    # P_D (no scaling) on the RT config too, and in-place application with batch 2
    w, od, gd = _both(3)
    r = synth.rhs(7, od.n_total, 2)
    P = fdp.build_block(gd)
    rt = dev(r)
    ws = P.workspace(2)
    P.apply(rt, rt, batch=2, workspace=ws)
    ref = oprec.BlockPrecond(od).apply(r)
    assert rel(rt.cpu().numpy(), ref) < TOL


def test_graph_replay_and_host_e2e():
    w, od, gd = _both(1)
    P = fdp.build_block(gd)
    rng = np.random.default_rng(3)
    ref = oprec.BlockPrecond(od)
    r1 = dev(rng.standard_normal(od.n_total))
    s1 = torch.empty_like(r1)
    ws = P.workspace(1)
    P.apply(r1, s1, workspace=ws)
    # same pointers -> graph replay with new contents
    r_new = rng.standard_normal(od.n_total)
    r1.copy_(dev(r_new))
    P.apply(r1, s1, workspace=ws)
    assert rel(s1.cpu().numpy(), ref.apply(r_new)) < TOL
    # host end-to-end path
    rh = rng.standard_normal(od.n_total)
    sh = np.zeros_like(rh)
    P.apply_host(rh, sh)
    assert rel(sh, ref.apply(rh)) < TOL


@pytest.mark.parametrize("cid,batch", [(1, 1), (2, 1), (3, 1), (1, 3), (3, 2)])
def test_host_e2e_pipeline(cid, batch):
    """block_precond_apply_host's copy/compute pipeline (per block at batch 1, per item above)
    with pinned (fdp.host_empty) and pageable buffers, repeated calls, vs the oracle."""
    w, od, gd = _both(cid)
    dv = dq = None
    if w.variable_nu:
        dv, dq = ospaces.nu_scalings(od, synth.viscosity)
    P = fdp.build_block(gd, dscale_vel=dv, dscale_pres=dq)
    ref = oprec.BlockPrecond(od, dv, dq)
    rng = np.random.default_rng(cid + 10 * batch)
    for pinned in (True, False):
        for _ in range(2):
            r = rng.standard_normal((batch, od.n_total))
            rh = fdp.host_empty(r.shape) if pinned else np.empty_like(r)
            rh[...] = r
            sh = fdp.host_empty(r.shape) if pinned else np.empty_like(r)
            P.apply_host(rh, sh, batch=batch)
            for b in range(batch):
                assert rel(sh[b], ref.apply(r[b])) < TOL


def test_errors_are_reported():
    w, od, gd = _both(1)
    P = fdp.build_block(gd)
    rh = np.zeros(od.n_total)
    with pytest.raises(fdp.FdpError) as e:
        import ctypes
        fdp._check(fdp.lib.block_precond_apply(P.h, ctypes.c_void_p(rh.ctypes.data),
                                               ctypes.c_void_p(rh.ctypes.data), 1,
                                               ctypes.c_void_p(rh.ctypes.data), None))
    assert e.value.status == 1  # FDP_ERR_INVALID_ARG: host pointer where device required
    # batch = 0 is a no-op
    fdp._check(fdp.lib.block_precond_apply(P.h, None, None, 0, None, None))


def test_fd_eigs_match_oracle_spectrum():
    K, M = fdp.iga_univariate(6, 4, 128, fdp.FDP_IGA_INTERIOR)
    S = fdp.FD([K, K, K], [M, M, M], (2, 1, 1))
    lam, U = S.get_eigs(0)
    lo, _ = ofd.gen_eig(K, M)
    assert np.max(np.abs(lam - lo)) / lo.max() < 1e-13
    assert np.max(np.abs(U.T @ M @ U - np.eye(len(lam)))) < 1e-11


@pytest.mark.slow
def test_block_precond_config4_full_size_bench_launch():
    """Config 4 at full size in the bench launch configuration (batch 8 in one call, the K1t
    folded transforms of DESIGN.md §5): all 8 items compared with the oracle element by element,
    per block, in relative L2 and max-abs (north_star: <= 1e-9)."""
    w, od, gd = _both(4)
    r = synth.rhs(w.seed, od.n_total, w.batch)
    P = fdp.build_block(gd)
    s = P.apply(dev(r), batch=w.batch)
    ref = oprec.BlockPrecond(od)
    o = od.offsets()
    for i in range(w.batch):
        si = s[i].cpu().numpy()
        ri = ref.apply(r[i])
        for k in range(len(o) - 1):
            assert rel(si[o[k]:o[k + 1]], ri[o[k]:o[k + 1]]) < TOL, (i, k)
            assert relmax(si[o[k]:o[k + 1]], ri[o[k]:o[k + 1]]) < TOL, (i, k)


@pytest.mark.slow
def test_config5_full_size_oracle_parity():
    """Config 5 (548.8 M dofs, RT p = 4, 512^3) at full size in the bench launch configuration:
    every block of the GPU apply against the oracle's Algorithm 1 (its own eigensolver, numpy
    mode products, banded pressure solve) element by element -- relative L2 and max-abs <= 1e-9
    (north_star). This covers the K1t tiles of n = 515 / 516 (odd-start mirror tiles, 4 column
    tiles of 9 / 8 n8 tiles) that the random-pencil cases reach only at smaller sizes."""
    w, od, gd = _both(5)
    b = synth.rhs(w.seed, od.n_total, 1)[0]
    P = fdp.build_block(gd)
    x = P.apply(dev(b)).cpu().numpy()
    del P
    torch.cuda.empty_cache()
    ref = oprec.BlockPrecond(od).apply(b)
    o = od.offsets()
    for k in range(len(o) - 1):
        assert rel(x[o[k]:o[k + 1]], ref[o[k]:o[k + 1]]) < TOL, k
        assert relmax(x[o[k]:o[k + 1]], ref[o[k]:o[k + 1]]) < TOL, k


@pytest.mark.parametrize("env", [{"FDP_NO_SMALL": "1"}, {"FDP_NO_FUSE": "1"}, {"FDP_PRESSURE": "banded"},
                                 {"FDP_PRESSURE": "dense"},
                                 {"FDP_NO_FOLD": "1"}, {"FDP_NO_PLANE": "1"}, {}])
@pytest.mark.parametrize("cfg_id", [1, 2, 3])
def test_block_precond_kernel_paths(cfg_id, env, monkeypatch):
    """Every kernel path (big/small K1, fused middle, banded/dense P_Q) against the oracle."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    w, od, gd = _both(cfg_id)
    r = synth.rhs(100 + cfg_id, od.n_total, 2)
    dv = dq = None
    if w.variable_nu:
        dv, dq = ospaces.nu_scalings(od, synth.viscosity)
    P = fdp.build_block(gd, dscale_vel=dv, dscale_pres=dq)
    s = P.apply(dev(r), batch=2).cpu().numpy()
    ref = oprec.BlockPrecond(od, dv, dq).apply(r)
    o = od.offsets()
    for i in range(2):
        for k in range(len(o) - 1):
            assert rel(s[i, o[k]:o[k + 1]], ref[i, o[k]:o[k + 1]]) < TOL, (cfg_id, env, k)


@pytest.mark.parametrize("dims", [(96, 5, 7), (8, 96, 33), (17, 3, 96), (9, 11), (65, 65, 65), (7, 9, 1),
                                  (3, 2, 40)])
def test_fd_apply_small_path_edges(dims):
    """n = 96 (largest small-path extent), tiny extents, 2D; fused middle + in-place pass 0,
    plane pipeline with a handle-owned counter set (max_batch = 3)."""
    rng = np.random.default_rng(sum(dims))
    Ks = [_rand_spd(n, rng, 1.0) for n in dims]
    Ms = [_rand_spd(n, rng, 2.0) for n in dims]
    coef = [1.0 + 0.5 * d for d in range(len(dims))]
    N = int(np.prod(dims))
    b = rng.standard_normal((3, N))
    S = fdp.FD(Ks, Ms, coef, max_batch=3)
    bt = dev(b)
    S.apply(bt, bt, batch=3)
    ref = ofd.FDSolver(Ks, Ms, coef)
    x = bt.cpu().numpy()
    for i in range(3):
        assert rel(x[i], ref.apply(b[i])) < TOL


def test_repeated_applies_and_batch_growth():
    """Many applies in a row on the same handle (graph replays), then a larger batch (a new
    captured graph and workspace)."""
    w, od, gd = _both(2)
    P = fdp.build_block(gd)
    ref = oprec.BlockPrecond(od)
    rng = np.random.default_rng(21)
    for batch in (1, 1, 3):
        r = rng.standard_normal((batch, od.n_total))
        rt = dev(r)
        st = torch.empty_like(rt)
        ws = P.workspace(batch)
        for _ in range(5):
            P.apply(rt, st, batch=batch, workspace=ws)
        s = st.cpu().numpy()
        for i in range(batch):
            assert rel(s[i], ref.apply(r[i])) < TOL


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("case", [(3, "RT", 2, 6), (3, "TH", 2, 5)])
def test_slab_decomposed_apply_emulated(G, case):
    """Config-5-style slab decomposition: G virtual ranks on one device (exchanges as device
    copies), libfdp's slab phases + pack/unpack kernels; result = oracle P_D^{-1} r."""
    from paper_1712_00403_b200 import dist as fdist
    D, disc, p, n_el = case
    od = ospaces.build(D, disc, p, n_el)
    gd = fdp.discretization(D, disc, p, n_el)
    P = fdp.build_block(gd)
    r = np.random.default_rng(G).standard_normal(od.n_total)
    s = fdist.emulate_slab_apply(P, dev(r), G).cpu().numpy()
    ref = oprec.BlockPrecond(od).apply(r)
    assert rel(s, ref) < TOL


@pytest.mark.parametrize("env", [{}, {"FDP_NO_SMALL": "1"}, {"FDP_NO_FUSE": "1"}])
def test_slab_decomposed_config3_size(env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    from paper_1712_00403_b200 import dist as fdist
    w, od, gd = _both(3)
    P = fdp.build_block(gd)
    r = synth.rhs(w.seed, od.n_total, 1)[0]
    s = fdist.emulate_slab_apply(P, dev(r), 8).cpu().numpy()
    ref = oprec.BlockPrecond(od).apply(r)
    assert rel(s, ref) < TOL


def test_slab_block_precond_nccl_single_rank():
    """SlabBlockPrecond through libfdp's NCCL communicator (fdp_nccl_unique_id broadcast over a
    torch.distributed group, fdp_comm_init, block_precond_apply_sharded: grouped phases, one
    grouped ncclSend/ncclRecv all-to-all per exchange). World size 1 on this box: the exchanges
    are NCCL self send/recv; multi-rank exchange counts are covered by tests/test_dist_cpu.py and
    the slab phases by the emulated-rank tests. Repeated, inside a CUDA graph, and with the
    block's P^G scalings (config 3, D_V = nu, D_Q = 1/nu)."""
    import os
    import socket
    import torch.distributed as tdist
    from paper_1712_00403_b200 import dist as fdist
    s0 = socket.socket()
    s0.bind(("127.0.0.1", 0))
    port = s0.getsockname()[1]
    s0.close()
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    created = False
    if not tdist.is_initialized():
        tdist.init_process_group("gloo", rank=0, world_size=1)
        created = True
    try:
        w, od, gd = _both(3)
        P = fdp.build_block(gd)
        SB = fdist.SlabBlockPrecond(P)
        assert SB.local_n == od.n_total
        ref = oprec.BlockPrecond(od)
        rng = np.random.default_rng(9)
        for _ in range(2):
            r = rng.standard_normal(od.n_total)
            rt = dev(r)
            st = torch.empty_like(rt)
            SB.apply(rt, st)
            assert rel(st.cpu().numpy(), ref.apply(r)) < TOL
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            SB.apply(rt, st)
        r = rng.standard_normal(od.n_total)
        rt.copy_(dev(r))
        g.replay()
        torch.cuda.synchronize()
        assert rel(st.cpu().numpy(), ref.apply(r)) < TOL
        del g  # a graph holding NCCL work must go before its communicator (ncclCommDestroy waits)
        torch.cuda.synchronize()
        SB.close()
        dv, dq = ospaces.nu_scalings(od, synth.viscosity)
        PG = fdp.build_block(gd, dscale_vel=dv, dscale_pres=dq)
        SG = fdist.SlabBlockPrecond(PG)
        SG.apply(rt, st)
        assert rel(st.cpu().numpy(), oprec.BlockPrecond(od, dv, dq).apply(r)) < TOL
        SG.close()
        # one FD solve through fd_apply_sharded, with a D scaling
        comp = od.comps[1]
        F = fdp.FD(gd.Ks[1], gd.Ms[1], gd.coef[1])
        SF = fdist.ShardedFD(F)
        N = int(np.prod(F.dims))
        b = rng.standard_normal(N)
        dsc = rng.uniform(0.5, 1.5, N)
        x = SF.apply(dev(b), torch.empty(N, dtype=torch.float64, device="cuda"),
                     dscale=dev(1.0 / np.sqrt(dsc))).cpu().numpy()
        xr = ofd.scaled_apply(ofd.FDSolver(comp.Ks, comp.Ms, comp.coef), b, dsc)
        assert rel(x, xr) < TOL and relmax(x, xr) < TOL
        SF.close()
    finally:
        if created:
            tdist.destroy_process_group()


def test_sharded_errors():
    """A peer-store communicator cannot serve fd_apply_sharded; bad communicator arguments are
    reported, not crashed on."""
    import ctypes
    rng = np.random.default_rng(3)
    F = fdp.FD([_rand_spd(n, rng, 1.0) for n in (9, 8, 7)], [_rand_spd(n, rng, 2.0) for n in (9, 8, 7)],
               (1.0, 1.0, 1.0))
    c = ctypes.c_void_p()
    uid = ctypes.create_string_buffer(128)
    assert fdp.lib.fdp_comm_init(1, 1, uid, 0, ctypes.byref(c)) == 1   # rank >= nranks
    assert fdp.lib.fdp_comm_init(1, 0, None, 0, ctypes.byref(c)) == 1
    assert fdp.lib.fd_sharded_workspace_bytes(F.h, None) == 0


@pytest.mark.parametrize("G", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("case", [(3, "RT", 2, 6), (3, "TH", 2, 5)])
@pytest.mark.parametrize("env", [{}, {"FDP_NO_SMALL": "1"}])
def test_slab_peer_store_emulated(G, case, env, monkeypatch):
    """Peer-store slab exchange (epilogue scatter into the owners' buffers) for G
    virtual ranks on one device (buffers poisoned with NaN: every element must be written
    exactly where the next phase reads it); small and big contraction paths."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    from paper_1712_00403_b200 import dist as fdist
    D, disc, p, n_el = case
    od = ospaces.build(D, disc, p, n_el)
    gd = fdp.discretization(D, disc, p, n_el)
    P = fdp.build_block(gd)
    r = np.random.default_rng(G).standard_normal(od.n_total)
    s = fdist.emulate_slab_apply_peer(P, dev(r), G).cpu().numpy()
    ref = oprec.BlockPrecond(od).apply(r)
    assert np.all(np.isfinite(s))
    assert rel(s, ref) < TOL


def test_slab_peer_store_config3_size():
    from paper_1712_00403_b200 import dist as fdist
    w, od, gd = _both(3)
    P = fdp.build_block(gd)
    r = synth.rhs(w.seed, od.n_total, 1)[0]
    s = fdist.emulate_slab_apply_peer(P, dev(r), 8).cpu().numpy()
    assert rel(s, oprec.BlockPrecond(od).apply(r)) < TOL


def test_peer_slab_block_precond_single_rank():
    """PeerSlabBlockPrecond through a real process group of one rank: IPC-allocated buffers,
    the peer-store phases and the system-scope barrier kernel (signalling itself), applied
    repeatedly (epoch counter) and captured in a CUDA graph."""
    import os
    import socket
    import torch.distributed as tdist
    from paper_1712_00403_b200 import dist as fdist
    s0 = socket.socket()
    s0.bind(("127.0.0.1", 0))
    port = s0.getsockname()[1]
    s0.close()
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    created = False
    if not tdist.is_initialized():
        tdist.init_process_group("gloo", rank=0, world_size=1)
        created = True
    try:
        w, od, gd = _both(3)
        P = fdp.build_block(gd)
        SB = fdist.PeerSlabBlockPrecond(P)
        ref = oprec.BlockPrecond(od)
        rng = np.random.default_rng(5)
        for _ in range(3):
            r = rng.standard_normal(od.n_total)
            rt = dev(r)
            st = torch.empty_like(rt)
            SB.apply(rt, st)
            assert rel(st.cpu().numpy(), ref.apply(r)) < TOL
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            SB.apply(rt, st)
        r = rng.standard_normal(od.n_total)
        rt.copy_(dev(r))
        for _ in range(2):
            g.replay()
        torch.cuda.synchronize()
        assert rel(st.cpu().numpy(), ref.apply(r)) < TOL
        SB.close()
        # P_D^G: the block's D scalings, sliced to the slab, inside block_precond_apply_sharded
        dv, dq = ospaces.nu_scalings(od, synth.viscosity)
        PG = fdp.build_block(gd, dscale_vel=dv, dscale_pres=dq)
        SG = fdist.PeerSlabBlockPrecond(PG)
        r = rng.standard_normal(od.n_total)
        rt = dev(r)
        SG.apply(rt, st)
        assert rel(st.cpu().numpy(), oprec.BlockPrecond(od, dv, dq).apply(r)) < TOL
        SG.close()
    finally:
        if created:
            tdist.destroy_process_group()


@pytest.mark.slow
def test_config5_full_size_residual():
    """Config 5 (548 M dofs) at full size in the bench launch configuration: a single output of
    an FD solve needs the whole solve, so the check is the property that holds at any size —
    the Sylvester residual ||R_k x_k - b_k|| / ||b_k|| of every velocity block (R_k applied by the
    oracle's Kronecker matvec with the oracle's own pencils) and ||P_Q x_p - b_p|| / ||b_p||
    of the pressure block. Bound: eps * kappa(R) ~ 1e-16 * 1e7 (SURVEY App. A spectra)."""
    from oracle import kron as okron
    w, od, gd = _both(5)
    b = synth.rhs(w.seed, od.n_total, 1)[0]
    P = fdp.build_block(gd)
    x = P.apply(dev(b)).cpu().numpy()
    o = od.offsets()
    for k, c in enumerate(od.comps):
        xk, bk = x[o[k]:o[k + 1]], b[o[k]:o[k + 1]]
        Rx = np.zeros_like(bk)
        for d in range(3):
            F = [c.Ks[e] if e == d else c.Ms[e] for e in range(3)]
            Rx += c.coef[d] * okron.kron_matvec(list(reversed(F)), xk)
        res = np.linalg.norm(Rx - bk) / np.linalg.norm(bk)
        assert res < 1e-9, (k, res)
        del Rx
    xp, bp = x[o[3]:], b[o[3]:]
    Mx = okron.kron_matvec(list(reversed(od.Mq)), xp)
    assert np.linalg.norm(Mx - bp) / np.linalg.norm(bp) < 1e-12


def test_empty_batches_are_noops():
    """batch = 0 (empty input) is a successful no-op for every apply entry point."""
    import ctypes
    w, od, gd = _both(1)
    P = fdp.build_block(gd)
    x = torch.full((od.n_total,), 7.0, dtype=torch.float64, device="cuda")
    ws = P.workspace(1)
    lib = fdp.lib
    assert lib.block_precond_apply(P.h, x.data_ptr(), x.data_ptr(), 0, ws.data_ptr(), None) == 0
    f = P.fds[0]
    assert lib.fd_apply(f.h, x.data_ptr(), x.data_ptr(), None, 0, ws.data_ptr(), None) == 0
    assert lib.kron_mass_apply(P.mass.h, 0, x.data_ptr(), x.data_ptr(), None, 0, None) == 0
    assert lib.block_precond_apply_host(P.h, ctypes.c_void_p(1), ctypes.c_void_p(1), 0, None) == 0
    torch.cuda.synchronize()
    assert torch.all(x == 7.0)


def test_config3_literal_c3_reading():
    """SURVEY.md C-3's secondary row: config 3 with the literal 'C^3' regularity in the RT own
    direction (130 x 68 x 68 per component at 64^3: the own-direction mode leaves the small
    path), P_D^G with the Greville scalings, against the oracle built the same way."""
    w = synth.CONFIGS[3]
    od = ospaces.build(w.dim, w.disc, w.p, w.n_el, rt_own_alpha=w.p - 1)
    gd = fdp.discretization(w.dim, w.disc, w.p, w.n_el, rt_own_alpha=w.p - 1)
    assert gd.comp_dims == [c.dims for c in od.comps] and gd.q_dims == od.q_dims
    assert gd.comp_dims[0] == [130, 68, 68] and od.n_total == 2117792
    dv, dq = ospaces.nu_scalings(od, synth.viscosity)
    gdv, gdq = fdp.nu_scalings(gd, synth.viscosity_separable(gd.D))
    assert np.max(np.abs(gdv - dv)) < 1e-14 and np.max(np.abs(gdq - dq)) < 1e-14
    P = fdp.build_block(gd, dscale_vel=dv, dscale_pres=dq)
    r = synth.rhs(w.seed, od.n_total, 1)
    s = P.apply(dev(r), batch=1).cpu().numpy()
    ref = oprec.BlockPrecond(od, dv, dq).apply(r)
    o = od.offsets()
    for k in range(len(o) - 1):
        assert rel(s[0, o[k]:o[k + 1]], ref[0, o[k]:o[k + 1]]) < TOL, k


@pytest.mark.parametrize("env", [{}, {"FDP_NO_FOLD": "1"}])
def test_block_precond_k1_sized_pressure(env, monkeypatch):
    """2D TH p=2 on 100 elements: velocity extents 200 (folded K1 transforms) and pressure
    extents 102 > 96, whose dense M_d^{-1} passes take the folded K1 FOLD_SYM kernel."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    od = ospaces.build(2, "TH", 2, 100)
    gd = fdp.discretization(2, "TH", 2, 100)
    assert gd.q_dims == [102, 102]
    P = fdp.build_block(gd)
    r = np.random.default_rng(31).standard_normal((2, od.n_total))
    s = P.apply(dev(r), batch=2).cpu().numpy()
    ref = oprec.BlockPrecond(od).apply(r)
    o = od.offsets()
    for i in range(2):
        for k in range(len(o) - 1):
            assert rel(s[i, o[k]:o[k + 1]], ref[i, o[k]:o[k + 1]]) < TOL, (env, k)


def relmax(a, b):
    """max |a - b| / max |b|: a single wrong element fails it even when the L2 norm hides it."""
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


@pytest.mark.parametrize("dims,coef,batch,dscale", [
    ((516, 9, 7), (2.0, 1.0, 1.0), 1, False),   # config 5's even extent in mode 1 (KMAJ K1t)
    ((516, 9, 7), (2.0, 1.0, 1.0), 2, True),    # ... batch 2, P^G (odd item stride: pad pass)
    ((7, 515, 9), (1.0, 2.0, 1.0), 1, True),    # config 5's odd extent in mode 2 (5-D maps)
    ((7, 515, 9), (1.0, 2.0, 1.0), 2, False),
    ((9, 7, 516), (1.0, 1.0, 2.0), 1, False),   # mode 3: Lambda epilogue on K1t
    ((9, 7, 516), (1.0, 1.0, 2.0), 3, True),
    ((259, 130, 97), (2.0, 1.0, 1.0), 2, True), # config 4's extent, odd n1 (pad pass), 3 folded K1 modes
    ((260, 131, 99), (1.0, 2.0, 1.0), 1, False),# even n1: the input read in place by TMA
    ((130, 300, 97), (1.0, 1.0, 2.0), 2, False),# several column tiles and p-groups, batch 2
    ((97, 2), (2.0, 1.0), 2, True),             # 2D, KMAJ only
])
def test_k1t_folded_transforms(dims, coef, batch, dscale):
    """K1t (TMA + mbarrier folded transform) on random persymmetric pencils whose
    folded modes exceed the small path: element-wise against the oracle's dense Algorithm 1
    (rel. L2 and max-abs <= 1e-9, north_star) and against the cp.async K1f path (FDP_NO_TMA=1,
    <= 1e-12); the TMA kernel must actually have run."""
    import os
    rng = np.random.default_rng(sum(dims) + 11 * batch)
    Ks = [_rand_persym_spd(n, rng, 1.0) for n in dims]
    Ms = [_rand_persym_spd(n, rng, 2.0) for n in dims]
    N = int(np.prod(dims))
    b = rng.standard_normal((batch, N))
    dsc = rng.uniform(0.5, 1.5, N) if dscale else None
    kw = {"dscale": dev(1.0 / np.sqrt(dsc))} if dscale else {}
    t0 = int(fdp.lib.fdp_debug_k1_launches(1))
    x = fdp.FD(Ks, Ms, coef).apply(dev(b), batch=batch, **kw).cpu().numpy()
    assert int(fdp.lib.fdp_debug_k1_launches(1)) > t0, "K1t did not run"
    os.environ["FDP_NO_TMA"] = "1"
    try:
        x_f = fdp.FD(Ks, Ms, coef).apply(dev(b), batch=batch, **kw).cpu().numpy()
    finally:
        del os.environ["FDP_NO_TMA"]
    ref = ofd.FDSolver(Ks, Ms, coef)
    for i in range(batch):
        r = ofd.scaled_apply(ref, b[i], dsc) if dscale else ref.apply(b[i])
        assert rel(x[i], r) < TOL and relmax(x[i], r) < TOL
        assert rel(x[i], x_f[i]) < 1e-12


def test_kron_mass_slab_workspace_covers_both_phases():
    """kron_mass_slab_workspace_bytes covers phase 0's z-slab and phase 1's y-slab (ADVICE r01:
    n2 != n3 with an uneven split, e.g. n2 = 11, n3 = 10, G = 2)."""
    rng = np.random.default_rng(3)
    dims = (4, 11, 10)
    Ms = [_rand_spd(n, rng, 2.0) for n in dims]
    Mb = fdp.KronMass(Ms)
    for G in (1, 2, 3):
        for rk in range(G):
            nb = int(fdp.lib.kron_mass_slab_workspace_bytes(Mb.h, G, rk))
            z = [10 // G + (1 if i < 10 % G else 0) for i in range(G)][rk]
            y = [11 // G + (1 if i < 11 % G else 0) for i in range(G)][rk]
            assert nb >= 8 * max(4 * 11 * z, 4 * y * 10), (G, rk, nb)


@pytest.mark.parametrize("G", [2, 3])
def test_slab_peer_store_k1t_scatter(G):
    """K1t's peer-store scatter: RT p = 4, n_el = 100 (component extents 103 / 104,
    all on the K1-path fold), G virtual ranks with NaN-poisoned receive buffers; the components
    with an even n1 run the scattering passes (phase 0's mode 2, phase 1's mode-3 backward) on
    K1t, the odd one on K1f. Against the oracle, every element."""
    from paper_1712_00403_b200 import dist as fdist
    od = ospaces.build(3, "RT", 4, 100)
    gd = fdp.discretization(3, "RT", 4, 100)
    P = fdp.build_block(gd)
    r = np.random.default_rng(50 + G).standard_normal(od.n_total)
    t0 = int(fdp.lib.fdp_debug_k1_launches(1))
    s = fdist.emulate_slab_apply_peer(P, dev(r), G).cpu().numpy()
    assert int(fdp.lib.fdp_debug_k1_launches(1)) > t0
    ref = oprec.BlockPrecond(od).apply(r)
    assert np.all(np.isfinite(s))
    assert rel(s, ref) < TOL and relmax(s, ref) < TOL
