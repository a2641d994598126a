"""Multi-GPU plumbing for the FD block preconditioner.

* Batch sharding (config 4): independent right-hand sides dealt round-robin to ranks; no
  collective in the apply (``batch_shard``).
* Slab decomposition (config 5): the slowest axis i3 of every block is partitioned over ranks;
  modes 1-2 run locally on i3-slabs, mode 3 on i2-slabs between two all-to-all exchanges
  (NCCL over NVLink / NVSwitch through ``torch.distributed``), computed by libfdp's slab phases
  (``fd_apply_slab`` / ``kron_mass_apply_slab``). The exchange plan below is pure index
  arithmetic; every floating-point operation runs in libfdp's kernels.

The same plan drives ``SlabBlockPrecond`` (one process per GPU) and ``emulate_slab_apply`` (all
ranks in one process on one device, exchanges as device copies) used by the single-GPU tests.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def part(n: int, G: int, r: int):
    """Even split of n over G ranks (first n mod G ranks own one more): (lo, len)."""
    q, rem = divmod(n, G)
    lo = r * q + min(r, rem)
    return lo, q + (1 if r < rem else 0)


def batch_shard(batch: int, world: int, rank: int):
    """Items {rank, rank + world, ...} of a batch (config 4's RHS sharding)."""
    return list(range(rank, batch, world))


@dataclass
class BlockPlan:
    """Exchange plan of one 3D block (n1, n2, n3) over G ranks, from rank g's point of view."""
    dims: tuple
    G: int
    g: int

    @property
    def z(self):
        return part(self.dims[2], self.G, self.g)

    @property
    def y(self):
        return part(self.dims[1], self.G, self.g)

    @property
    def zslab_size(self):
        n1, n2, _ = self.dims
        return n1 * n2 * self.z[1]

    @property
    def yslab_size(self):
        n1, _, n3 = self.dims
        return n1 * self.y[1] * n3

    def ex1_splits(self):
        """(send sizes, recv sizes) of exchange 1 (piece buffer -> y-slab), in rank order."""
        n1, n2, n3 = self.dims
        nz = self.z[1]
        ny = self.y[1]
        send = [n1 * part(n2, self.G, h)[1] * nz for h in range(self.G)]
        recv = [n1 * ny * part(n3, self.G, h)[1] for h in range(self.G)]
        return send, recv

    def ex2_splits(self):
        """(send sizes, recv sizes) of exchange 2 (y-slab -> piece buffer)."""
        s, r = self.ex1_splits()
        return r, s

    def zslab_offset(self):
        """Offset of this rank's z-slab in the full (unsharded) block vector."""
        n1, n2, _ = self.dims
        return n1 * n2 * self.z[0]


def nccl_comm(group=None, device: int = 0):
    """A libfdp NCCL communicator over a torch.distributed group (fdp_comm_init): rank 0 of the
    group draws the ncclUniqueId (fdp_nccl_unique_id), the group broadcasts its 128 bytes
    (torch.distributed is plumbing here), every rank initialises. Returns the fdp_comm handle."""
    import ctypes

    import torch.distributed as dist
    from . import _check, lib

    G, g = dist.get_world_size(group), dist.get_rank(group)
    uid = ctypes.create_string_buffer(128)
    if g == 0:
        _check(lib.fdp_nccl_unique_id(uid))
    box = [uid.raw if g == 0 else None]
    dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0,
                               group=group)
    uid = ctypes.create_string_buffer(box[0], 128)
    c = ctypes.c_void_p()
    _check(lib.fdp_comm_init(G, g, uid, device, ctypes.byref(c)))
    return c


class SlabBlockPrecond:
    """P_D^{-1} (or (P_D^G)^{-1} with the block's own scalings) with every block slab-decomposed
    over a torch.distributed process group, exchanges through libfdp's NCCL communicator
    (fdp_comm_init + block_precond_apply_sharded: all blocks' phases as grouped launches, one
    grouped NCCL send/recv all-to-all per exchange). The local vector layout is
    [u_1 z-slab | ... | u_D z-slab | p z-slab]. D = 3 only."""

    def __init__(self, block, group=None):
        import torch
        import torch.distributed as dist
        from . import lib

        self.torch = torch
        self.group = group
        self.G = dist.get_world_size(group)
        self.g = dist.get_rank(group)
        self.block = block
        self.fds = block.fds
        self.mass = block.mass
        self.plans = [BlockPlan(tuple(f.dims), self.G, self.g) for f in self.fds]
        self.plans.append(BlockPlan(tuple(self.mass.dims), self.G, self.g))
        self.local_sizes = [p.zslab_size for p in self.plans]
        self.local_off = np.concatenate([[0], np.cumsum(self.local_sizes)]).astype(np.int64)
        self.local_n = int(self.local_off[-1])
        assert self.local_n == int(lib.block_precond_sharded_size(block.h, self.G, self.g))
        self.comm = nccl_comm(group, block.device)
        wsb = int(lib.block_precond_sharded_workspace_bytes(block.h, self.comm))
        self.ws = torch.empty(wsb // 8 + 1, dtype=torch.float64, device=f"cuda:{block.device}")

    def apply(self, r, s, stream=None):
        from . import _check, _dev, _stream, lib
        _check(lib.block_precond_apply_sharded(self.block.h, self.comm, _dev(r, "r", self.local_n),
                                               _dev(s, "s", self.local_n), _dev(self.ws, "workspace"),
                                               _stream(stream)))
        return s

    def close(self):
        from . import lib
        if getattr(self, "comm", None):
            lib.fdp_comm_destroy(self.comm)
            self.comm = None


class ShardedFD:
    """One FD solve slab-decomposed over a process group (fd_apply_sharded, NCCL communicator):
    x = D^{-1/2} U Lambda^{-1} U^T D^{-1/2} b on this rank's z-slab (planes
    slab_range(n3, G, g) of the vec-ordered tensor)."""

    def __init__(self, fd, group=None):
        import torch
        import torch.distributed as dist
        from . import lib

        self.fd = fd
        self.G, self.g = dist.get_world_size(group), dist.get_rank(group)
        self.plan = BlockPlan(tuple(fd.dims), self.G, self.g)
        self.local_n = self.plan.zslab_size
        self.comm = nccl_comm(group, fd.device)
        wsb = int(lib.fd_sharded_workspace_bytes(fd.h, self.comm))
        self.ws = torch.empty(wsb // 8 + 1, dtype=torch.float64, device=f"cuda:{fd.device}")

    def apply(self, b, x, dscale=None, stream=None):
        from . import _check, _dev, _stream, lib
        _check(lib.fd_apply_sharded(self.fd.h, self.comm, _dev(b, "b", self.local_n), _dev(x, "x", self.local_n),
                                    None if dscale is None else _dev(dscale, "dscale", self.local_n),
                                    _dev(self.ws, "workspace"), _stream(stream)))
        return x

    def close(self):
        from . import lib
        if getattr(self, "comm", None):
            lib.fdp_comm_destroy(self.comm)
            self.comm = None


def emulate_slab_apply(block, r_full, G: int):
    """Run the slab-decomposed application for G virtual ranks in one process on one device,
    performing the two exchanges as device copies. Returns the full result vector (torch)."""
    import torch
    from . import fd_apply_slab, kron_mass_apply_slab, lib

    dev = r_full.device
    blocks = [("fd", f, tuple(f.dims)) for f in block.fds] + [("mass", block.mass, tuple(block.mass.dims))]
    full_off = np.concatenate([[0], np.cumsum([int(np.prod(b[2])) for b in blocks])]).astype(np.int64)
    out = torch.empty_like(r_full)
    for bi, (kind, h, dims) in enumerate(blocks):
        plans = [BlockPlan(dims, G, g) for g in range(G)]
        base = int(full_off[bi])
        wsb = max((lib.fd_slab_workspace_bytes(h.h, G, g) if kind == "fd"
                   else lib.kron_mass_slab_workspace_bytes(h.h, G, g)) for g in range(G))
        ws = torch.empty(wsb // 8 + 1, dtype=torch.float64, device=dev)
        run = fd_apply_slab if kind == "fd" else kron_mass_apply_slab
        sends = []
        for g, p in enumerate(plans):
            zo = base + p.zslab_offset()
            xs = r_full[zo:zo + p.zslab_size].contiguous()
            snd = torch.empty(p.zslab_size, dtype=torch.float64, device=dev)
            run(h, 0, G, g, xs, snd, None, ws)
            sends.append(snd)
        # exchange 1: rank g's y-slab = concatenation over sources h of piece g of h's send buffer
        ybufs = []
        for g, p in enumerate(plans):
            pieces = []
            for hsrc in range(G):
                ssz, _ = plans[hsrc].ex1_splits()
                off = int(np.sum(ssz[:g]))
                pieces.append(sends[hsrc][off:off + ssz[g]])
            yb = torch.cat(pieces).contiguous()
            assert yb.numel() == p.yslab_size
            run(h, 1, G, g, yb, yb, None, ws if kind == "fd" else None)
            ybufs.append(yb)
        # exchange 2: rank g receives from every h the planes of g's z-range of h's y-slab
        for g, p in enumerate(plans):
            pieces = []
            for hsrc in range(G):
                ssz, _ = plans[hsrc].ex2_splits()
                off = int(np.sum(ssz[:g]))
                pieces.append(ybufs[hsrc][off:off + ssz[g]])
            rc = torch.cat(pieces).contiguous()
            xs = torch.empty(p.zslab_size, dtype=torch.float64, device=dev)
            run(h, 2, G, g, rc, xs, None, ws if kind == "fd" else None)
            zo = base + p.zslab_offset()
            out[zo:zo + p.zslab_size] = xs
    return out


# ------------------------------------------------------------------------------------------------
# Peer-store exchange: the exchanges fused into the contraction epilogues
# ------------------------------------------------------------------------------------------------
def allgather_bytes(blob: bytes, group=None) -> list:
    """Every rank's byte string, in rank order (torch.distributed all_gather_object: host-side
    plumbing for the IPC handle blobs of the peer-store exchange)."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(blob), group=group)
    return out


class PeerSlabBlockPrecond:
    """P_D^{-1} slab-decomposed over a process group with the peer-store exchange, through
    libfdp's communicator (fdp_comm_create / fdp_comm_connect / block_precond_apply_sharded):
    every rank owns, per block, a y-slab receive buffer and a z-slab return buffer mapped into
    every peer (CUDA IPC); phase 0's mode-2 epilogue and phase 1's last mode-3 epilogue store
    straight into the owners' buffers over NVLink, and a system-scope barrier kernel separates the
    phases. No pack / unpack kernels, no NCCL call in the apply. This class only moves the IPC
    handle blobs between ranks (torch.distributed all_gather_object). Local layout as
    SlabBlockPrecond: [u_1 z-slab | ... | u_D z-slab | p z-slab]. D = 3 only."""

    def __init__(self, block, group=None):
        import ctypes

        import torch
        import torch.distributed as dist
        from . import _check, lib

        self.torch = torch
        self.G = G = dist.get_world_size(group)
        self.g = g = dist.get_rank(group)
        self.block = block
        self.fds = block.fds
        self.mass = block.mass
        self.plans = [BlockPlan(tuple(f.dims), G, g) for f in self.fds]
        self.plans.append(BlockPlan(tuple(self.mass.dims), G, g))
        self.local_sizes = [p.zslab_size for p in self.plans]
        self.local_off = np.concatenate([[0], np.cumsum(self.local_sizes)]).astype(np.int64)
        self.local_n = int(self.local_off[-1])
        assert self.local_n == int(lib.block_precond_sharded_size(block.h, G, g))
        nb = int(lib.fdp_comm_blob_bytes(block.h, G))
        blob = ctypes.create_string_buffer(nb)
        c = ctypes.c_void_p()
        _check(lib.fdp_comm_create(block.h, G, g, ctypes.byref(c), blob))
        self.comm = c
        blobs = allgather_bytes(blob.raw, group)
        allb = ctypes.create_string_buffer(b"".join(blobs), nb * G)
        _check(lib.fdp_comm_connect(c, allb))
        wsb = int(lib.block_precond_sharded_workspace_bytes(block.h, c))
        self.ws = torch.empty(wsb // 8 + 1, dtype=torch.float64, device=f"cuda:{block.device}")
        dist.barrier(group)

    def apply(self, r, s, stream=None):
        from . import _check, _dev, _stream, lib
        _check(lib.block_precond_apply_sharded(self.block.h, self.comm, _dev(r, "r", self.local_n),
                                               _dev(s, "s", self.local_n), _dev(self.ws, "workspace"),
                                               _stream(stream)))
        return s

    def close(self):
        from . import lib
        if getattr(self, "comm", None):
            lib.fdp_comm_destroy(self.comm)
            self.comm = None


def emulate_slab_apply_peer(block, r_full, G: int):
    """The peer-store phases for G virtual ranks in one process on one device: every rank's
    receive buffers are local tensors and the 'peers' arrays point at them, so the epilogue
    scatter runs exactly as across GPUs; the phases run rank after rank (no barrier kernel: a
    sequential schedule already orders them). Returns the full result vector (torch)."""
    import torch
    from . import fd_apply_slab_peer, kron_mass_apply_slab_peer, lib

    dev = r_full.device
    blocks = [("fd", f, tuple(f.dims)) for f in block.fds] + [("mass", block.mass, tuple(block.mass.dims))]
    full_off = np.concatenate([[0], np.cumsum([int(np.prod(b[2])) for b in blocks])]).astype(np.int64)
    out = torch.empty_like(r_full)
    for bi, (kind, h, dims) in enumerate(blocks):
        plans = [BlockPlan(dims, G, g) for g in range(G)]
        base = int(full_off[bi])
        wsb = max((lib.fd_slab_workspace_bytes(h.h, G, g) if kind == "fd"
                   else lib.kron_mass_slab_workspace_bytes(h.h, G, g)) for g in range(G))
        ws = torch.empty(wsb // 8 + 1, dtype=torch.float64, device=dev)
        run = fd_apply_slab_peer if kind == "fd" else kron_mass_apply_slab_peer
        ybuf = [torch.full((max(p.yslab_size, 1),), float("nan"), dtype=torch.float64, device=dev) for p in plans]
        zbuf = [torch.full((max(p.zslab_size, 1),), float("nan"), dtype=torch.float64, device=dev) for p in plans]
        py = torch.tensor([t.data_ptr() for t in ybuf], dtype=torch.int64, device=dev)
        pz = torch.tensor([t.data_ptr() for t in zbuf], dtype=torch.int64, device=dev)
        for g, p in enumerate(plans):
            zo = base + p.zslab_offset()
            xs = r_full[zo:zo + p.zslab_size].contiguous()
            if p.zslab_size:
                run(h, 0, G, g, xs, None, py, None, ws)
        for g, p in enumerate(plans):
            if p.yslab_size:
                run(h, 1, G, g, ybuf[g], None, pz, None, ws)
        for g, p in enumerate(plans):
            if p.zslab_size:
                xs = torch.empty(p.zslab_size, dtype=torch.float64, device=dev)
                run(h, 2, G, g, zbuf[g], xs, None, None, ws)
                zo = base + p.zslab_offset()
                out[zo:zo + p.zslab_size] = xs
        torch.cuda.synchronize()
    return out
