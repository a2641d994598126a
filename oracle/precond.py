"""Block preconditioners of PAPER.md §4: block-diagonal P_D = diag(P_V,1, .., P_V,D, P_Q)
(§5, §6), block-triangular P_T and constrained P_C.
Oracle only (test infrastructure; imported by tests/, __graft_entry__.smoke() and bench.py's
reference leg, never by the product path)."""
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

    def apply_vel(self, ru: np.ndarray) -> np.ndarray:
        """P_V^{-1} r_u = (P_V,1^{-1} r_1, .., P_V,D^{-1} r_D) on the velocity part [r_1 | .. | r_D]."""
        s = np.empty_like(ru)
        o = self.off
        for k, solver in enumerate(self.vel):
            sl = slice(o[k], o[k + 1])
            dk = None if self.dv is None else self.dv[o[k]:o[k + 1]]
            s[sl] = fd.scaled_apply(solver, ru[sl], dk)
        return s

    def apply_pres(self, rp: np.ndarray) -> np.ndarray:
        """P_Q^{-1} r_p."""
        return self.pres.scaled_inverse(rp, self.dq)

    def apply(self, r: np.ndarray) -> np.ndarray:
        r = np.asarray(r, dtype=np.float64)
        if r.ndim == 2:
            return np.stack([self.apply(row) for row in r])
        nv = self.off[-2]
        return np.concatenate([self.apply_vel(r[:nv]), self.apply_pres(r[nv:])])


class TriangularPrecond:
    """Block upper-triangular P_T = [[P_V, B^T], [0, -P_Q]] (§4 eq. (P_T), P:603-611;
    P_T^G with the geometry/diagonal-scaled blocks). Back substitution:
    s_p = -P_Q^{-1} r_p, then s_u = P_V^{-1} (r_u - B^T s_p). ``stokes`` supplies B^T
    (StokesCube.BT_apply)."""

    def __init__(self, block: BlockPrecond, stokes):
        self.block = block
        self.stokes = stokes
        self.nv = block.off[-2]

    def apply(self, r: np.ndarray) -> np.ndarray:
        ru, rp = r[:self.nv], r[self.nv:]
        sp_ = -self.block.apply_pres(rp)
        su = self.block.apply_vel(ru - self.stokes.BT_apply(sp_))
        return np.concatenate([su, sp_])


class ConstrainedPrecond:
    """Constrained P_C = [[P_V, B^T], [B, B P_V^{-1} B^T - P_Q]], applied through the
    paper's factorization, right to left:
    P_C^{-1} = [[I, -P_V^{-1} B^T], [0, I]] . diag(I, -P_Q^{-1}) . [[I, 0], [-B, I]] . diag(P_V^{-1}, I)."""

    def __init__(self, block: BlockPrecond, stokes):
        self.block = block
        self.stokes = stokes
        self.nv = block.off[-2]

    def apply(self, r: np.ndarray) -> np.ndarray:
        ru, rp = r[:self.nv], r[self.nv:]
        u = self.block.apply_vel(ru)                                 # diag(P_V^{-1}, I)
        p = rp - self.stokes.B_apply(u)                              # [[I, 0], [-B, I]]
        p = -self.block.apply_pres(p)                                # diag(I, -P_Q^{-1})
        u = u - self.block.apply_vel(self.stokes.BT_apply(p))        # [[I, -P_V^{-1} B^T], [0, I]]
        return np.concatenate([u, p])
