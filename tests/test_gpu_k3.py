"""K3t (kernels/kron_mass.cu mass_tile_kernel): the banded pressure solve P_Q^{-1} b (PAPER.md
P:975-976, per-mode application) with each tile of 16 fibers solved in shared memory,
against the oracle's Kronecker mass inverse element by element (relative L2 and max-abs <= 1e-9).

The cases reach the tile kernel in mode 1 (fiber-major tiles, even n) and modes >= 2 (row tiles,
even P), ragged last tiles (P % 16 != 0), recurrence lengths with n % 4 != 0 (the single-step
tails), band 1..5, batch > 1 with the batch stride, the P^G scaling, in-place calls, and the
fall-backs to the sweep kernels (odd extents, tiles above the shared-memory limit)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1712_00403_b200 as fdp  # noqa: E402
from oracle import mass as omass  # noqa: E402
from oracle import univariate  # noqa: E402

pytestmark = pytest.mark.gpu
TOL = 1e-9


def _check(x, ref):
    x, ref = np.asarray(x), np.asarray(ref)
    rl2 = np.linalg.norm(x - ref) / np.linalg.norm(ref)
    mx = np.max(np.abs(x - ref)) / np.max(np.abs(ref))
    assert rl2 <= TOL and mx <= TOL, (rl2, mx)


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("pn,batch", [
    (((4, 512), (4, 6), (4, 4)), 1),     # config 5's pressure extent in mode 1; P = 516 ragged tiles
    (((3, 127), (2, 33), (5, 20)), 2),   # n = 130 (n % 4 = 2), odd n in mode 2, batch stride
    (((3, 30), (4, 8), (2, 8)), 1),      # odd n1 and odd P in mode 2: sweep kernels, mode 3 tiles
    (((1, 41), (1, 13), (2, 5)), 3),     # band 1
    (((5, 40), (5, 11), (5, 9)), 1),     # band 5
    (((2, 1798), (2, 4), (1, 3)), 1),    # n = 1800: tiles above the shared-memory limit (sweeps)
    (((2, 1698), (2, 4), (1, 3)), 1),    # n = 1700: the largest tiles that fit
    (((4, 60), (4, 28)), 2),             # 2D
])
def test_k3_tile_inverse_vs_oracle(pn, batch):
    rng = np.random.default_rng(31)
    Ms = [univariate.pressure_mass(p, ne) for p, ne in pn]
    km = omass.KronMass(Ms)
    N = int(np.prod(km.dims))
    b = rng.standard_normal((batch, N))
    dq = rng.uniform(0.5, 2.0, N)
    K = fdp.KronMass(Ms)
    x = K.apply(dev(b), batch=batch).cpu().numpy()
    z = K.apply(dev(b), dscale=dev(1 / np.sqrt(dq)), batch=batch).cpu().numpy()
    bi = dev(b)
    K.apply(bi, bi, batch=batch)  # in place
    xi = bi.cpu().numpy()
    for i in range(batch):
        ref = km.inverse(b[i])
        _check(x[i], ref)
        _check(xi[i], ref)
        _check(z[i], km.scaled_inverse(b[i], dq))


def test_k3_tile_config5_pressure_sampled_fibers():
    """Config 5's pressure block (516^3, p = 4, the bench launch) on sampled whole fibers: the
    Kronecker inverse applied to e_j (x) e_k (x) v has the closed form
    (M_3^{-1} e_k) (x) (M_2^{-1} e_j) (x) (M_1^{-1} v), so rank-1 inputs check every mode's tiles
    at full size against three dense univariate solves."""
    M = univariate.pressure_mass(4, 512)
    n = M.shape[0]
    K = fdp.KronMass([M, M, M])
    rng = np.random.default_rng(5)
    v = rng.standard_normal(n)
    Minv = np.linalg.inv(M)
    for (j, k) in [(0, 0), (3, 515), (257, 100)]:
        a2 = np.zeros(n); a2[j] = 1.0
        a3 = np.zeros(n); a3[k] = 1.0
        b = torch.zeros(n, n, n, dtype=torch.float64, device="cuda")  # [i3, i2, i1]
        b[k, j, :] = dev(v)
        x = K.apply(b.reshape(-1)).reshape(n, n, n)
        y1, y2, y3 = Minv @ v, Minv @ a2, Minv @ a3
        for (i3, i2) in [(0, 0), (k, j), (515, 2), (100, 257)]:
            ref = y3[i3] * y2[i2] * y1
            got = x[i3, i2, :].cpu().numpy()
            assert np.max(np.abs(got - ref)) <= TOL * np.max(np.abs(y3)) * np.max(np.abs(y2)) * np.max(np.abs(y1))
        # the i1 = 7 plane holds y1[7] * (y3 (x) y2)
        plane = x[:, :, 7].cpu().numpy()
        _check(plane, y1[7] * np.outer(y3, y2))


# K3u (mass_utile_kernel): the persistent 4-warp kernel with the coefficient rows in shared memory
# and right-looking substitutions; taken when n % 4 == 0, n >= 16, band <= 5 (mode 1: any fiber
# count; modes >= 2: even P). The cases cover both tile layouts, ragged last tiles (fiber counts and
# P not multiples of 12), several tiles per warp (the mbarrier phase flips), band 1..5, batch > 1,
# the P^G scaling and in-place calls.
K3U_CASES = [
    (((4, 512), (4, 12), (4, 16)), 1),    # n = 516, 16, 20: config 5's extent in mode 1
    (((2, 62), (2, 126), (2, 126)), 1),   # 1366 / 768 / 683 tiles on 592 warps: 2-3 tiles per warp
    (((3, 25), (2, 30), (1, 19)), 2),     # n = 28, 32, 20: P = 28 ragged p-blocks, mixed bands, batch
    (((1, 39), (1, 15), (1, 19)), 3),     # band 1
    (((5, 35), (5, 15), (5, 11)), 1),     # band 5 (the forward window spans two groups)
    (((4, 60), (4, 28)), 2),              # 2D
    (((4, 252), (4, 20)), 1),             # 2D, n = 256: whole groups only, P = 256 ragged (21 x 12 + 4)
]


@pytest.mark.parametrize("pn,batch", K3U_CASES)
def test_k3u_inverse_vs_oracle(pn, batch):
    test_k3_tile_inverse_vs_oracle(pn, batch)


def test_k3t_cases_with_k3u_disabled():
    """FDP_K3_U is read once per process: re-run the K3t and K3u cases in a child with K3u off, so
    the K3t tile kernel and the sweeps stay covered on the shapes K3u now takes."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FDP_K3_U="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", os.path.abspath(__file__),
                        "-k", "inverse_vs_oracle or sampled_fibers"], cwd=root, env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
