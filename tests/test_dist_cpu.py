"""Multi-process (world size 2, gloo, CPU) tests of the multi-GPU host logic:
the slab-decomposition exchange plan of paper_1712_00403_b200.dist with real all_to_all_single
exchanges, the piece-buffer layout libfdp's pack/unpack kernels implement (restated here in
numpy), and the whole sharded FD application with the oracle doing the local mode products.
Also the batch sharding of config 4."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1712_00403_b200 import dist as fdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _pack(zslab, plan):
    """Piece-buffer layout of include/fdp.h: piece h = [i3 local][i2 - y0_h][i1] at n1*nz*y0_h."""
    n1, n2, _ = plan.dims
    G = plan.G
    Z = zslab.reshape((n1, n2, -1), order="F")
    out = []
    for h in range(G):
        y0, ny = fdist.part(n2, G, h)
        out.append(np.reshape(Z[:, y0:y0 + ny, :], -1, order="F"))
    return np.concatenate(out)


def _unpack(pieces, plan):
    n1, n2, _ = plan.dims
    nz = plan.z[1]
    Z = np.zeros((n1, n2, nz))
    off = 0
    for h in range(plan.G):
        y0, ny = fdist.part(n2, plan.G, h)
        sz = n1 * ny * nz
        Z[:, y0:y0 + ny, :] = np.reshape(pieces[off:off + sz], (n1, ny, nz), order="F")
        off += sz
    return np.reshape(Z, -1, order="F")


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _run(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    return res


def _exchange_roundtrip(rank, world):
    dims = (5, 7, 9)
    full = np.random.default_rng(0).standard_normal(int(np.prod(dims)))
    T = full.reshape(dims, order="F")
    plan = fdist.BlockPlan(dims, world, rank)
    z0, nz = plan.z
    y0, ny = plan.y
    zslab = np.reshape(T[:, :, z0:z0 + nz], -1, order="F")
    send = torch.from_numpy(_pack(zslab, plan))
    s1, r1 = plan.ex1_splits()
    ybuf = torch.empty(sum(r1), dtype=torch.float64)
    dist.all_to_all_single(ybuf, send, output_split_sizes=r1, input_split_sizes=s1)
    expect_y = np.reshape(T[:, y0:y0 + ny, :], -1, order="F")
    ok1 = np.array_equal(ybuf.numpy(), expect_y)
    s2, r2 = plan.ex2_splits()
    back = torch.empty(sum(r2), dtype=torch.float64)
    dist.all_to_all_single(back, ybuf, output_split_sizes=r2, input_split_sizes=s2)
    ok2 = np.array_equal(_unpack(back.numpy(), plan), zslab)
    return bool(ok1 and ok2)


def _sharded_fd(rank, world):
    from oracle import fd, kron, univariate
    Kn, Mn = univariate.rt_normal_pencil(2, 4)
    Kt, Mt = univariate.rt_tangential_pencil(2, 4)
    Ks, Ms = [Kt, Kn, Kt], [Mt, Mn, Mt]   # component 2 of an RT space: (6, 5, 6)
    coef = (1.0, 2.0, 1.0)
    S = fd.FDSolver(Ks, Ms, coef)
    dims = tuple(K.shape[0] for K in Ks)
    b = np.random.default_rng(1).standard_normal(int(np.prod(dims)))
    plan = fdist.BlockPlan(dims, world, rank)
    z0, nz = plan.z
    y0, ny = plan.y
    B = b.reshape(dims, order="F")[:, :, z0:z0 + nz]
    # modes 1, 2 forward locally
    B = kron.mode_product(kron.mode_product(B, S.Us[0].T, 1), S.Us[1].T, 2)
    send = torch.from_numpy(_pack(np.reshape(B, -1, order="F"), plan))
    s1, r1 = plan.ex1_splits()
    ybuf = torch.empty(sum(r1), dtype=torch.float64)
    dist.all_to_all_single(ybuf, send, output_split_sizes=r1, input_split_sizes=s1)
    Y = ybuf.numpy().reshape((dims[0], ny, dims[2]), order="F")
    Y = kron.mode_product(Y, S.Us[2].T, 3) / S.Lam[:, y0:y0 + ny, :]
    Y = kron.mode_product(Y, S.Us[2], 3)
    s2, r2 = plan.ex2_splits()
    back = torch.empty(sum(r2), dtype=torch.float64)
    dist.all_to_all_single(back, torch.from_numpy(np.reshape(Y, -1, order="F").copy()),
                           output_split_sizes=r2, input_split_sizes=s2)
    X = _unpack(back.numpy(), plan).reshape((dims[0], dims[1], nz), order="F")
    X = kron.mode_product(kron.mode_product(X, S.Us[1], 2), S.Us[0], 1)
    ref = S.apply(b).reshape(dims, order="F")[:, :, z0:z0 + nz]
    return float(np.max(np.abs(X - ref)) / np.max(np.abs(ref)))


def _exchange_roundtrip_libfdp(rank, world):
    """The exchange plan of libfdp's NCCL sharded apply (fdp_slab_exchange_counts: the per-peer
    counts its grouped ncclSend / ncclRecv use, pieces at cumulative offsets) driven through real
    all-to-alls: exchange 1 must deliver exactly the y-slab, exchange 2 the packed z-slab back."""
    import paper_1712_00403_b200 as fdp
    ok = True
    for dims in ((5, 7, 9), (4, 3, 10), (6, 11, 2)):
        full = np.random.default_rng(sum(dims)).standard_normal(int(np.prod(dims)))
        T = full.reshape(dims, order="F")
        plan = fdist.BlockPlan(dims, world, rank)
        z0, nz = plan.z
        y0, ny = plan.y
        zslab = np.reshape(T[:, :, z0:z0 + nz], -1, order="F")
        s1, r1 = fdp.slab_exchange_counts(dims, world, rank, 1)
        s2, r2 = fdp.slab_exchange_counts(dims, world, rank, 2)
        ybuf = torch.empty(sum(r1), dtype=torch.float64)
        dist.all_to_all_single(ybuf, torch.from_numpy(_pack(zslab, plan)), output_split_sizes=r1,
                               input_split_sizes=s1)
        ok = ok and np.array_equal(ybuf.numpy(), np.reshape(T[:, y0:y0 + ny, :], -1, order="F"))
        back = torch.empty(sum(r2), dtype=torch.float64)
        dist.all_to_all_single(back, ybuf, output_split_sizes=r2, input_split_sizes=s2)
        ok = ok and np.array_equal(_unpack(back.numpy(), plan), zslab)
    return bool(ok)


def test_libfdp_exchange_counts_roundtrip_gloo():
    for world in (2, 3):
        res = _run(_exchange_roundtrip_libfdp, world)
        assert res == {r: True for r in range(world)}, res


@pytest.mark.parametrize("dims", [(5, 7, 9), (515, 516, 516), (133, 133, 133), (3, 2, 1)])
@pytest.mark.parametrize("G", [1, 2, 3, 8])
def test_libfdp_exchange_counts_match_plan(dims, G):
    """fdp_slab_exchange_counts agrees with the Python BlockPlan for every rank, and exchange 2 is
    exchange 1 reversed; the counts conserve the z-slab and the y-slab."""
    import paper_1712_00403_b200 as fdp
    for g in range(G):
        plan = fdist.BlockPlan(dims, G, g)
        s1, r1 = fdp.slab_exchange_counts(dims, G, g, 1)
        s2, r2 = fdp.slab_exchange_counts(dims, G, g, 2)
        assert (s1, r1) == tuple(plan.ex1_splits()) and (s2, r2) == tuple(plan.ex2_splits())
        assert sum(s1) == plan.zslab_size and sum(r1) == plan.yslab_size


def test_slab_exchange_roundtrip_gloo():
    res = _run(_exchange_roundtrip)
    assert res == {0: True, 1: True}


def test_sharded_fd_matches_oracle_gloo():
    res = _run(_sharded_fd)
    for r in (0, 1):
        assert isinstance(res[r], float) and res[r] < 1e-13, res


@pytest.mark.parametrize("n,G", [(516, 8), (515, 8), (7, 3), (5, 8), (133, 4)])
def test_part_covers_axis(n, G):
    spans = [fdist.part(n, G, r) for r in range(G)]
    assert spans[0][0] == 0
    assert all(a + l == spans[i + 1][0] for i, (a, l) in enumerate(spans[:-1]))
    assert spans[-1][0] + spans[-1][1] == n
    assert max(l for _, l in spans) - min(l for _, l in spans) <= 1


def test_batch_shard_config4():
    for world in (1, 2, 4, 8):
        shards = [fdist.batch_shard(8, world, r) for r in range(world)]
        assert sorted(sum(shards, [])) == list(range(8))
        assert len(set(len(s) for s in shards)) == 1


def _handles(rank, world):
    blob = bytes([rank, 7]) * 160  # stand-in for a rank's blob of 64-byte IPC handles
    allb = fdist.allgather_bytes(blob)
    return all(allb[r] == bytes([r, 7]) * 160 for r in range(world))


def test_peer_handle_exchange_gloo():
    """The host plumbing of the peer-store exchange (PeerSlabBlockPrecond): every rank gets every
    rank's IPC handle blob, in rank order (world size 2, gloo)."""
    res = _run(_handles)
    assert res == {0: True, 1: True}
