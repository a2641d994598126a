"""Block-diagonal preconditioner P_D = diag(P_V,1, .., P_V,D, P_Q) (§4 P:591-598,
§5, §6). Oracle only."""
from __future__ import annotations

import numpy as np

from . import fd, mass, spaces


class BlockPrecond:
    """P_D^{-1} r = (P_V,1^{-1} r_1, .., P_V,D^{-1} r_D, P_Q^{-1} r_p);
    with dscales, the P_D^G variant D^{-1/2} P^{-1} D^{-1/2} blockwise."""

    def __init__(self, disc: spaces.Discretization, dscale_vel=None, dscale_pres=None):
        self.disc = disc
        self.vel = [fd.FDSolver(c.Ks, c.Ms, c.coef) for c in disc.comps]
        self.pres = mass.KronMass(disc.Mq)
        self.off = disc.offsets()
        self.dv = dscale_vel
        self.dq = dscale_pres

    def apply(self, r: np.ndarray) -> np.ndarray:
        r = np.asarray(r, dtype=np.float64)
        if r.ndim == 2:
            return np.stack([self.apply(row) for row in r])
        s = np.empty_like(r)
        o = self.off
        for k, solver in enumerate(self.vel):
            sl = slice(o[k], o[k + 1])
            dk = None if self.dv is None else self.dv[o[k]:o[k + 1]]
            s[sl] = fd.scaled_apply(solver, r[sl], dk)
        sl = slice(o[-2], o[-1])
        s[sl] = self.pres.scaled_inverse(r[sl], self.dq)
        return s
