"""Small applies of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck, one tool per gpurun call): config 1 (2D plane kernel), config 2 (mode-1 passes + 3D
plane kernel, P_Q alongside), config 3 with P^G scalings, the K1t TMA kernel on small persymmetric
pencils (KMAJ with the odd-start fix-up box, 5-D maps, Lambda and scale epilogues, pad pass), the
cp.async K1f path (FDP_NO_TMA), the banded pressure solve (K3), the emulated peer-store slab phases
and the real one-rank peer-store path (IPC buffers + system-scope barrier kernel). Diagnostic only:
prints one line per case and exits non-zero on the first failure."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1712_00403_b200 as fdp
import synth


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def persym_spd(n, rng, shift):
    a = rng.standard_normal((n, n))
    a = a @ a.T + shift * n * np.eye(n)
    j = a[::-1, ::-1]
    return 0.5 * (a + j)


def block_case(cid, batch=1, scaled=False):
    w = synth.CONFIGS[cid]
    gd = fdp.discretization(w.dim, w.disc, w.p, w.n_el)
    kw = {}
    if scaled:
        rng = np.random.default_rng(5)
        kw = {"dscale_vel": rng.uniform(0.5, 1.5, sum(gd.sizes[:-1])),
              "dscale_pres": rng.uniform(0.5, 1.5, gd.sizes[-1])}
    P = fdp.build_block(gd, **kw)
    r = dev(np.random.default_rng(cid).standard_normal((batch, gd.n_total)))
    s = P.apply(r, batch=batch)
    torch.cuda.synchronize()
    assert torch.isfinite(s).all()
    P.close()
    print("ok block", cid, batch, scaled, flush=True)


def fd_case(dims, coef, batch, dscale, env=None):
    env = env or {}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        rng = np.random.default_rng(sum(dims))
        Ks = [persym_spd(n, rng, 1.0) for n in dims]
        Ms = [persym_spd(n, rng, 2.0) for n in dims]
        N = int(np.prod(dims))
        b = dev(rng.standard_normal((batch, N)))
        kw = {"dscale": dev(rng.uniform(0.5, 1.5, N))} if dscale else {}
        F = fdp.FD(Ks, Ms, coef)
        x = F.apply(b, batch=batch, **kw)
        torch.cuda.synchronize()
        assert torch.isfinite(x).all()
        F.close()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    print("ok fd", dims, batch, dscale, env, flush=True)


def mass_case():
    os.environ["FDP_PRESSURE"] = "banded"
    try:
        block_case(2)
    finally:
        del os.environ["FDP_PRESSURE"]
    print("ok banded pressure", flush=True)


def slab_case():
    from paper_1712_00403_b200 import dist as fdist
    gd = fdp.discretization(3, "TH", 2, 5)
    P = fdp.build_block(gd)
    r = dev(np.random.default_rng(3).standard_normal(gd.n_total))
    for G in (1, 3):
        s = fdist.emulate_slab_apply_peer(P, r, G)
        assert torch.isfinite(s).all()
        s = fdist.emulate_slab_apply(P, r, G)
        assert torch.isfinite(s).all()
    print("ok slab emulated", flush=True)


def peer_case():
    import socket
    import torch.distributed as tdist
    from paper_1712_00403_b200 import dist as fdist
    s0 = socket.socket()
    s0.bind(("127.0.0.1", 0))
    port = s0.getsockname()[1]
    s0.close()
    tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        gd = fdp.discretization(3, "RT", 2, 6)
        P = fdp.build_block(gd)
        sp = fdist.PeerSlabBlockPrecond(P)
        r = dev(np.random.default_rng(4).standard_normal(sp.local_n))
        s = torch.empty_like(r)
        for _ in range(3):
            sp.apply(r, s)
        torch.cuda.synchronize()
        assert torch.isfinite(s).all()
        sp.close()
    finally:
        tdist.destroy_process_group()
    print("ok peer one rank", flush=True)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    cases = {
        "blocks": lambda: (block_case(1), block_case(2), block_case(3, scaled=True), block_case(2, batch=2)),
        "k1t": lambda: (fd_case((516, 9, 7), (2.0, 1.0, 1.0), 1, False),
                        fd_case((7, 515, 9), (1.0, 2.0, 1.0), 2, True),
                        fd_case((9, 7, 516), (1.0, 1.0, 2.0), 1, True),
                        fd_case((259, 130, 97), (2.0, 1.0, 1.0), 2, True),
                        fd_case((97, 2), (2.0, 1.0), 2, True)),
        "k1f": lambda: (fd_case((259, 130, 97), (2.0, 1.0, 1.0), 1, True, {"FDP_NO_TMA": "1"}),
                        fd_case((130, 300, 9), (1.0, 2.0, 1.0), 1, False, {"FDP_NO_TMA": "1"})),
        "mass": mass_case,
        "slab": slab_case,
        "peer": peer_case,
    }
    for name, fn in cases.items():
        if which in ("all", name):
            fn()
    print("all ok", flush=True)
