"""Fast Diagonalization direct solver (§5.2, Algorithm 1). Oracle only."""
from __future__ import annotations

import numpy as np
import scipy.linalg

from . import kron


def gen_eig(K: np.ndarray, M: np.ndarray):
    """Step 1: K U = M U D with U^T M U = I, eigenvalues ascending.

    LAPACK generalized symmetric-definite eigensolver as one library step. Signs are
    normalised so the largest-magnitude entry of each column is positive (cosmetic;
    x does not depend on it).
    """
    lam, U = scipy.linalg.eigh(K, M)
    idx = np.argmax(np.abs(U), axis=0)
    sgn = np.sign(U[idx, np.arange(U.shape[1])])
    sgn[sgn == 0] = 1.0
    return lam, U * sgn


def lambda_tensor(lams, coef) -> np.ndarray:
    """Lambda = sum_d c_d (I (x) .. (x) D_d (x) .. (x) I) as a tensor:
    Lambda[i1,..,iD] = sum_d c_d lambda_d[i_d] (c_d from P:678-688)."""
    D = len(lams)
    L = np.zeros(tuple(len(l) for l in lams))
    for d in range(D):
        shape = [1] * D
        shape[d] = len(lams[d])
        L = L + coef[d] * np.reshape(lams[d], shape)
    return L


class FDSolver:
    """R^{-1} for R = sum_d c_d (F_D (x) .. (x) F_1), F_d = K_d at position d and M_d elsewhere
    (coefficients P:678-688). Pencils are given per direction d = 1..D (index i_d)."""

    def __init__(self, Ks, Ms, coef):
        self.D = len(Ks)
        self.dims = [K.shape[0] for K in Ks]
        self.coef = [float(c) for c in coef]
        eig = [gen_eig(K, M) for K, M in zip(Ks, Ms)]
        self.lams = [e[0] for e in eig]
        self.Us = [e[1] for e in eig]
        self.Lam = lambda_tensor(self.lams, self.coef)
        lam_min = sum(c * l.min() for c, l in zip(self.coef, self.lams))
        lam_max = sum(c * l.max() for c, l in zip(self.coef, self.lams))
        if not lam_min > 1e-12 * lam_max:
            raise np.linalg.LinAlgError("singular Kronecker sum")

    def apply(self, t: np.ndarray) -> np.ndarray:
        """Algorithm 1 steps 2-4 with U = U_D (x) .. (x) U_1:
        t~ = t x_1 U_1^T .. x_D U_D^T;  q~ = t~ / Lambda;  q = q~ x_1 U_1 .. x_D U_D."""
        T = kron.unvec(t, self.dims)
        for d in range(self.D):
            T = kron.mode_product(T, self.Us[d].T, d + 1)
        Q = T / self.Lam
        for d in range(self.D):
            Q = kron.mode_product(Q, self.Us[d], d + 1)
        return kron.vec(Q)


def assemble_R(Ks, Ms, coef) -> np.ndarray:
    """Dense R = sum_d c_d (F_D (x) .. (x) F_1) for brute-force checks on tiny grids."""
    D = len(Ks)
    R = 0.0
    for d in range(D):
        F = [Ks[e] if e == d else Ms[e] for e in range(D)]
        R = R + coef[d] * kron.kron_dense(list(reversed(F)))
    return R


def dense_solve(Ks, Ms, coef, t: np.ndarray) -> np.ndarray:
    """The plain definition x = R^{-1} t by dense Cholesky."""
    R = assemble_R(Ks, Ms, coef)
    c = scipy.linalg.cho_factor(R)
    return scipy.linalg.cho_solve(c, t)


def scaled_apply(solver: FDSolver, t: np.ndarray, dscale: np.ndarray | None) -> np.ndarray:
    """P^G = D^{1/2} P D^{1/2}  =>  x = D^{-1/2} P^{-1} D^{-1/2} t (C-5)."""
    if dscale is None:
        return solver.apply(t)
    s = 1.0 / np.sqrt(dscale)
    return s * solver.apply(s * t)
