"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the paper's method: only the raw workload parameters
of BASELINE.json's five configs, the seeded N(0,1) right-hand-side generator and the
viscosity field of config 3. Each side (``oracle/`` and ``paper_1712_00403_b200``)
derives space dimensions, matrices, scalings and results on its own.

Recipe: the preconditioner input in the paper is a MINRES
residual of the driven cavity; FD is a dense direct method whose
cost and rounding behaviour do not depend on the data, so white noise
``numpy.random.default_rng(seed).standard_normal`` stands in.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = ["Workload", "CONFIGS", "rhs", "viscosity", "viscosity_separable"]


@dataclass(frozen=True)
class Workload:
    """Raw parameters of one BASELINE.json config (no derived quantities)."""

    name: str
    dim: int          # spatial dimension D (2 or 3)
    disc: str         # "TH" (Taylor-Hood) or "RT" (Raviart-Thomas)
    p: int            # pressure degree; velocity degree p+1
    n_el: int         # elements per parametric direction
    seed: int         # RHS seed
    batch: int        # independent right-hand sides
    variable_nu: bool  # config 3: diagonal scaling from nu(x) sampled at dofs


# BASELINE.json "configs", in order. alpha = p - 1 everywhere.
CONFIGS = {
    1: Workload("cfg1_2d_th_p2_16", 2, "TH", 2, 16, 0, 1, False),
    2: Workload("cfg2_3d_th_p3_32", 3, "TH", 3, 32, 1, 1, False),
    3: Workload("cfg3_3d_rt_p4_64_nu", 3, "RT", 4, 64, 2, 1, True),
    4: Workload("cfg4_3d_th_p5_128_b8", 3, "TH", 5, 128, 3, 8, False),
    5: Workload("cfg5_3d_rt_p4_512", 3, "RT", 4, 512, 4, 1, False),
}


def rhs(seed: int, n_total: int, batch: int = 1) -> np.ndarray:
    """FP64 N(0,1) right-hand side(s), shape (batch, n_total), row-major, one generator.

    Layout of each row is [u_1 | ... | u_D | p], each block in vec order (i1 fastest,
    PAPER.md P:382-386); the caller supplies n_total.
    """
    g = np.random.default_rng(seed)
    return g.standard_normal((batch, n_total), dtype=np.float64)


def viscosity(x, y, z=None):
    """Config 3 viscosity nu(x) = 1 + 0.5 sin(2 pi x) sin(2 pi y) sin(2 pi z) in [0.5, 1.5]."""
    s = np.sin(2 * math.pi * np.asarray(x)) * np.sin(2 * math.pi * np.asarray(y))
    if z is not None:
        s = s * np.sin(2 * math.pi * np.asarray(z))
    return 1.0 + 0.5 * s


def viscosity_separable(dim: int = 3):
    """The same nu as ``viscosity`` written as separable terms [(c_t, [w_t1(x), .., w_tD(x)])]:
    1 + 0.5 prod_d sin(2 pi x_d) (None = constant-1 term)."""
    s = lambda x: np.sin(2 * math.pi * np.asarray(x))
    return [(1.0, None), (0.5, [s] * dim)]
