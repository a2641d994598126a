"""GMRES (Saad & Schultz 1986, cited at PAPER.md P:619 for the P_T- and P_C-preconditioned solves;
tolerance 1e-8 and zero initial guess). Oracle harness only (test infrastructure).

Readings (G-1): full (unrestarted) GMRES with LEFT preconditioning, the Arnoldi process
by modified Gram-Schmidt and the least-squares problem by Givens rotations, exactly as in Saad &
Schultz's Algorithm; stop when the preconditioned residual ||P^{-1}(b - A x_k)|| relative to
||P^{-1} b|| is <= tol (the MATLAB gmres convention the paper's experiments ran under).
"""
from __future__ import annotations

import numpy as np


def gmres(matvec, b, precond, tol=1e-8, maxit=1000):
    """Solve A x = b; returns (x, iterations, history of ||z_k|| / ||z_0||), z = P^{-1} residual."""
    z = precond(np.asarray(b, dtype=np.float64))
    beta = float(np.linalg.norm(z))
    n = z.shape[0]
    if beta == 0.0:
        return np.zeros(n), 0, [0.0]
    m = min(maxit, n)
    V = np.zeros((m + 1, n))
    H = np.zeros((m + 1, m))
    cs = np.zeros(m)
    sn = np.zeros(m)
    g = np.zeros(m + 1)
    g[0] = beta
    V[0] = z / beta
    hist = [1.0]
    k = 0
    for j in range(m):
        w = precond(matvec(V[j]))
        for i in range(j + 1):                   # modified Gram-Schmidt
            H[i, j] = float(np.dot(w, V[i]))
            w = w - H[i, j] * V[i]
        H[j + 1, j] = float(np.linalg.norm(w))
        if H[j + 1, j] != 0.0:
            V[j + 1] = w / H[j + 1, j]
        for i in range(j):                       # previous rotations on the new column
            t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
            H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
            H[i, j] = t
        den = np.hypot(H[j, j], H[j + 1, j])
        cs[j] = H[j, j] / den
        sn[j] = H[j + 1, j] / den
        H[j, j] = den
        H[j + 1, j] = 0.0
        g[j + 1] = -sn[j] * g[j]
        g[j] = cs[j] * g[j]
        k = j + 1
        hist.append(abs(g[j + 1]) / beta)
        if abs(g[j + 1]) / beta <= tol or H[j, j] == 0.0:
            break
    y = np.zeros(k)
    for i in range(k - 1, -1, -1):               # back substitution R y = g
        y[i] = (g[i] - H[i, i + 1:k] @ y[i + 1:k]) / H[i, i]
    x = V[:k].T @ y
    return x, k, hist
