"""Kronecker pressure mass P_Q = M_D (x) .. (x) M_1 and its inverse.
Oracle only."""
from __future__ import annotations

import numpy as np
import scipy.linalg

from . import kron


def bandwidth(M: np.ndarray) -> int:
    """Half bandwidth of a symmetric matrix (number of non-zero super-diagonals)."""
    n = M.shape[0]
    for b in range(n - 1, 0, -1):
        if np.any(np.diagonal(M, b) != 0.0):
            return b
    return 0


def _upper_band(M: np.ndarray, b: int) -> np.ndarray:
    """LAPACK upper banded storage ab[b + i - j, j] = M[i, j]."""
    n = M.shape[0]
    ab = np.zeros((b + 1, n))
    for k in range(b + 1):
        ab[b - k, k:] = np.diagonal(M, k)
    return ab


class KronMass:
    """(M_D (x) .. (x) M_1)^{-1} via (A (x) B (x) C)^{-1} vec(X) = vec(X x_1 C^{-1} x_2 B^{-1}
    x_3 A^{-1}) with banded Cholesky of each univariate factor."""

    def __init__(self, Ms):
        self.Ms = [np.asarray(M, dtype=np.float64) for M in Ms]
        self.dims = [M.shape[0] for M in Ms]
        self.bands = [bandwidth(M) for M in self.Ms]
        self.chol = [scipy.linalg.cholesky_banded(_upper_band(M, b), lower=False)
                     for M, b in zip(self.Ms, self.bands)]

    def _solve_mode(self, X: np.ndarray, d: int) -> np.ndarray:
        Xd = np.moveaxis(X, d, 0)
        sh = Xd.shape
        Y = scipy.linalg.cho_solve_banded((self.chol[d], False), Xd.reshape(sh[0], -1))
        return np.moveaxis(Y.reshape(sh), 0, d)

    def inverse(self, t: np.ndarray) -> np.ndarray:
        X = kron.unvec(t, self.dims)
        for d in range(len(self.dims)):
            X = self._solve_mode(X, d)
        return kron.vec(X)

    def forward(self, t: np.ndarray) -> np.ndarray:
        """(M_D (x) .. (x) M_1) t."""
        return kron.kron_matvec(list(reversed(self.Ms)), t)

    def scaled_inverse(self, t: np.ndarray, dscale: np.ndarray | None) -> np.ndarray:
        """(P_Q^G)^{-1} t = D_Q^{-1/2} P_Q^{-1} D_Q^{-1/2} t."""
        if dscale is None:
            return self.inverse(t)
        s = 1.0 / np.sqrt(dscale)
        return s * self.inverse(s * t)
