"""Pins for oracle/fd.py: generalized eigenpairs and Algorithm 1 against brute force, closed
forms and special cases."""
import numpy as np
import pytest

from oracle import fd, kron, univariate


def _rand_spd(n, rng, shift=1.0):
    A = rng.standard_normal((n, n))
    return A @ A.T + shift * n * np.eye(n)


@pytest.mark.parametrize("p,n_el", [(2, 6), (3, 32), (4, 16)])
def test_gen_eig_m_orthonormal_and_residual(p, n_el):
    K, M = univariate.th_velocity_pencil(p, n_el)
    lam, U = fd.gen_eig(K, M)
    assert np.max(np.abs(U.T @ M @ U - np.eye(len(lam)))) < 1e-12
    assert np.max(np.abs(K @ U - M @ U * lam)) < 1e-12 * np.max(np.abs(K)) * 10
    assert np.all(np.diff(lam) >= 0)


def test_gen_eig_p1_dirichlet_closed_form():
    # p = 1 interior pencil: lambda_j = (6/h^2)(1 - cos(j pi h)) / (2 + cos(j pi h)), j = 1..n_el-1
    n_el = 10
    h = 1.0 / n_el
    K, M = univariate.stiffness_mass(1, 0, n_el)
    lam, U = fd.gen_eig(univariate.interior(K), univariate.interior(M))
    j = np.arange(1, n_el)
    exact = (6 / h**2) * (1 - np.cos(j * np.pi * h)) / (2 + np.cos(j * np.pi * h))
    assert np.max(np.abs(lam - exact) / exact) < 1e-13


def test_p1_fd_is_dst1():
    # Lynch-Rice-Thomas special case cited at P:979-980: eigenvectors are sine modes.
    n_el = 9
    h = 1.0 / n_el
    K, M = univariate.stiffness_mass(1, 0, n_el)
    lam, U = fd.gen_eig(univariate.interior(K), univariate.interior(M))
    i = np.arange(1, n_el)
    for j in range(1, n_el):
        s = np.sin(i * j * np.pi * h)
        u = U[:, j - 1]
        c = (u @ s) / (s @ s)
        assert np.max(np.abs(u - c * s)) < 1e-12 * np.max(np.abs(u))


def test_lambda_min_near_pi_squared():
    # lambda_min -> pi^2 for Dirichlet and Nitsche pencils of the configs
    for K, M in [univariate.th_velocity_pencil(3, 32), univariate.rt_tangential_pencil(4, 64),
                 univariate.rt_normal_pencil(4, 64)]:
        lam, _ = fd.gen_eig(K, M)
        assert abs(lam[0] - np.pi**2) < 0.05


@pytest.mark.parametrize("dims,coef", [((3, 4, 5), (2.0, 1.0, 1.0)), ((5, 3, 4), (1.0, 2.0, 1.0)),
                                        ((4, 5, 3), (1.0, 1.0, 2.0)), ((4, 6), (2.0, 1.0)),
                                        ((6, 4), (1.0, 2.0)), ((3, 4, 5), (0.7, 1.3, 2.9))])
def test_fd_equals_dense_solve_random_pencils(dims, coef):
    rng = np.random.default_rng(sum(dims))
    Ks = [_rand_spd(n, rng) for n in dims]
    Ms = [_rand_spd(n, rng, 2.0) for n in dims]
    t = rng.standard_normal(int(np.prod(dims)))
    x = fd.FDSolver(Ks, Ms, coef).apply(t)
    xd = fd.dense_solve(Ks, Ms, coef, t)
    assert np.linalg.norm(x - xd) / np.linalg.norm(xd) < 1e-12


def test_fd_equals_dense_solve_bspline_pencils_anisotropic():
    # mixed RT-like pencils with distinct sizes so that a wrong factor/index pairing fails
    Kn, Mn = univariate.rt_normal_pencil(2, 2)        # 3
    Kt, Mt = univariate.rt_tangential_pencil(2, 2)    # 4
    Kh, Mh = univariate.th_velocity_pencil(1, 3)      # 5
    Ks, Ms = [Kn, Kt, Kh], [Mn, Mt, Mh]
    rng = np.random.default_rng(3)
    t = rng.standard_normal(3 * 4 * 5)
    for coef in [(2, 1, 1), (1, 2, 1), (1, 1, 2)]:
        x = fd.FDSolver(Ks, Ms, coef).apply(t)
        xd = fd.dense_solve(Ks, Ms, coef, t)
        assert np.linalg.norm(x - xd) / np.linalg.norm(xd) < 1e-12


def test_fd_sylvester_residual_config2_component():
    K, M = univariate.th_velocity_pencil(3, 32)
    coef = (1.0, 2.0, 1.0)
    S = fd.FDSolver([K] * 3, [M] * 3, coef)
    b = np.random.default_rng(1).standard_normal(65**3)
    x = S.apply(b)
    # R x via Kronecker matvecs, never forming R
    Rx = sum(coef[d] * kron.kron_matvec(list(reversed([K if e == d else M for e in range(3)])), x)
             for d in range(3))
    assert np.linalg.norm(Rx - b) / np.linalg.norm(b) < 1e-10


def test_fd_symmetric_positive():
    K, M = univariate.th_velocity_pencil(2, 5)
    S = fd.FDSolver([K] * 3, [M] * 3, (2, 1, 1))
    rng = np.random.default_rng(5)
    s, t = rng.standard_normal((2, K.shape[0] ** 3))
    assert abs(t @ S.apply(s) - s @ S.apply(t)) < 1e-12 * abs(t @ S.apply(s)) + 1e-14
    assert t @ S.apply(t) > 0


def test_fd_identity_pencils():
    # K_d = M_d = I  =>  R = (sum c) I  =>  x = b / sum c
    dims = (3, 4, 2)
    Is = [np.eye(n) for n in dims]
    b = np.random.default_rng(2).standard_normal(24)
    x = fd.FDSolver(Is, Is, (2, 1, 1)).apply(b)
    assert np.max(np.abs(x - b / 4.0)) < 1e-15


def test_fd_scaled_constant_d():
    K, M = univariate.th_velocity_pencil(2, 4)
    S = fd.FDSolver([K] * 2, [M] * 2, (2, 1))
    b = np.random.default_rng(4).standard_normal(K.shape[0] ** 2)
    x1 = S.apply(b)
    x2 = fd.scaled_apply(S, b, np.full(b.shape, 4.0))
    assert np.max(np.abs(x2 - x1 / 4.0)) < 1e-15 * np.max(np.abs(x1)) * 10


def test_fd_singular_guard():
    with pytest.raises(np.linalg.LinAlgError):
        fd.FDSolver([np.diag([1e-20, 1.0])] * 2, [np.eye(2)] * 2, (1, 1))
