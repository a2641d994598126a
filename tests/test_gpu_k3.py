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
