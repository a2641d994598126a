"""Preconditioned MINRES (Paige & Saunders 1975, cited at PAPER.md P:600; tolerance 1e-8 and zero
initial guess). Oracle harness only (test infrastructure).

Stopping rule: the recurrence's preconditioned residual norm
phibar_k = ||r_k||_{P^{-1}} relative to phibar_0 <= tol. The preconditioner is any SPD
``apply(r) -> P^{-1} r`` callable, so the same code runs with the oracle's P_D or the GPU's.
"""
from __future__ import annotations

import numpy as np


def minres(matvec, b, precond, tol=1e-8, maxit=20000):
    """Returns (x, iterations, history of phibar/beta1)."""
    n = b.shape[0]
    x = np.zeros(n)
    r1 = b.copy()
    y = precond(r1)
    beta1 = float(np.dot(r1, y))
    if beta1 < 0:
        raise ValueError("preconditioner is not positive definite")
    beta1 = np.sqrt(beta1)
    if beta1 == 0.0:
        return x, 0, [0.0]
    oldb, beta, dbar, epsln, phibar = 0.0, beta1, 0.0, 0.0, beta1
    cs, sn = -1.0, 0.0
    w = np.zeros(n)
    w2 = np.zeros(n)
    r2 = r1.copy()
    hist = [1.0]
    eps = np.finfo(np.float64).eps
    for itn in range(1, maxit + 1):
        s = 1.0 / beta
        v = s * y
        y = matvec(v)
        if itn >= 2:
            y = y - (beta / oldb) * r1
        alfa = float(np.dot(v, y))
        y = y - (alfa / beta) * r2
        r1 = r2
        r2 = y
        y = precond(r2)
        oldb = beta
        beta = float(np.dot(r2, y))
        if beta < 0:
            raise ValueError("preconditioner is not positive definite")
        beta = np.sqrt(beta)
        oldeps = epsln
        delta = cs * dbar + sn * alfa
        gbar = sn * dbar - cs * alfa
        epsln = sn * beta
        dbar = -cs * beta
        gamma = max(np.hypot(gbar, beta), eps)
        cs = gbar / gamma
        sn = beta / gamma
        phi = cs * phibar
        phibar = sn * phibar
        w1 = w2
        w2 = w
        w = (v - oldeps * w1 - delta * w2) / gamma
        x = x + phi * w
        hist.append(phibar / beta1)
        if phibar / beta1 <= tol:
            return x, itn, hist
    return x, maxit, hist
