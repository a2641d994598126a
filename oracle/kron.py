"""Kronecker algebra (§2.3). Oracle only.

Tensors are numpy arrays of shape (n_1, ..., n_D) whose vec is Fortran order: vec index
i = i1 + (i2-1) n1 + (i3-1) n1 n2, i1 fastest.
"""
from __future__ import annotations

from functools import reduce

import numpy as np


def unvec(x: np.ndarray, dims) -> np.ndarray:
    """vec^{-1}: vector -> tensor with i1 fastest."""
    return np.reshape(x, tuple(dims), order="F")


def vec(W: np.ndarray) -> np.ndarray:
    """vec(W) with i1 fastest."""
    return np.reshape(W, -1, order="F")


def mode_product(W: np.ndarray, Y: np.ndarray, mode: int) -> np.ndarray:
    """m-mode product [W x_m Y]_{..i_m..} = sum_k Y[i_m, k] W[..k..], mode 1-based."""
    ax = mode - 1
    out = np.tensordot(Y, W, axes=([1], [ax]))  # new axis 0 = i_m
    return np.moveaxis(out, 0, ax)


def kron_dense(factors_slowest_first) -> np.ndarray:
    """Dense A_D (x) ... (x) A_1; the LAST factor acts on the fastest index i1."""
    return reduce(np.kron, factors_slowest_first)


def kron_matvec(factors_slowest_first, x: np.ndarray) -> np.ndarray:
    """(A_D (x) ... (x) A_1) vec(X) = vec(X x_1 A_1 ... x_D A_D) (P:414-418 with C-1's pairing:
    the factor written last in the Kronecker product acts on i1)."""
    A = list(reversed(factors_slowest_first))  # A[0] acts on i1
    dims = [a.shape[1] for a in A]
    X = unvec(x, dims)
    for d, a in enumerate(A):
        X = mode_product(X, a, d + 1)
    return vec(X)
