"""TH / RT discrete spaces of a workload: per-component pencils, coefficients, dims and the
config-3 diagonal scalings (§2.2, §5, §7). Oracle only.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import splines, univariate


@dataclass
class Component:
    Ks: list          # per direction d = 1..D (acts on index i_d)
    Ms: list
    coef: list        # c_d = 1 + [d = k]  (T_k = I + e_k e_k^T)
    grev: list        # Greville abscissae of the component's dofs per direction (C-6)

    @property
    def dims(self):
        return [K.shape[0] for K in self.Ks]

    @property
    def size(self):
        return int(np.prod(self.dims))


@dataclass
class Discretization:
    D: int
    disc: str
    p: int
    n_el: int
    comps: list       # velocity components k = 1..D
    Mq: list          # pressure mass factors per direction
    grev_q: list

    @property
    def q_dims(self):
        return [M.shape[0] for M in self.Mq]

    @property
    def sizes(self):
        return [c.size for c in self.comps] + [int(np.prod(self.q_dims))]

    @property
    def n_total(self):
        return int(sum(self.sizes))

    def offsets(self):
        return np.concatenate([[0], np.cumsum(self.sizes)]).astype(np.int64)


def _grev(deg, alpha, n_el, interior):
    g = splines.greville(splines.open_uniform_knots(deg, alpha, n_el), deg)
    return g[1:-1] if interior else g


def build(D: int, disc: str, p: int, n_el: int, rt_own_alpha: int | None = None) -> Discretization:
    """alpha = p - 1, p = pressure degree; TH velocity S^{p+1}_alpha restricted
    to interior functions in every direction; RT component k: S^{p+1}_{alpha+1}
    interior in direction k, S^p_alpha full elsewhere with Nitsche.
    rt_own_alpha: regularity of the RT own direction (default alpha + 1 = p, the paper;
    p - 1 is config 3's literal "C^3" wording)."""
    alpha = p - 1
    comps = []
    if disc == "TH":
        K, M = univariate.th_velocity_pencil(p, n_el)
        g = _grev(p + 1, alpha, n_el, True)
        for k in range(D):
            comps.append(Component([K] * D, [M] * D, [1.0 + (d == k) for d in range(D)], [g] * D))
    elif disc == "RT":
        Kn, Mn = univariate.rt_normal_pencil(p, n_el, rt_own_alpha)
        Kt, Mt = univariate.rt_tangential_pencil(p, n_el)
        gn = _grev(p + 1, alpha + 1 if rt_own_alpha is None else rt_own_alpha, n_el, True)
        gt = _grev(p, alpha, n_el, False)
        for k in range(D):
            comps.append(Component([Kn if d == k else Kt for d in range(D)],
                                   [Mn if d == k else Mt for d in range(D)],
                                   [1.0 + (d == k) for d in range(D)],
                                   [gn if d == k else gt for d in range(D)]))
    else:
        raise ValueError(disc)
    Mq = univariate.pressure_mass(p, n_el)
    gq = _grev(p, alpha, n_el, False)
    return Discretization(D, disc, p, n_el, comps, [Mq] * D, [gq] * D)


def _grid_eval(f, grevs):
    """f at the tensor grid of Greville points, returned in vec order (i1 fastest)."""
    G = np.meshgrid(*grevs, indexing="ij")
    return np.reshape(f(*G), -1, order="F")


def nu_scalings(disc: Discretization, nu):
    """Config 3's literal reading: D_V[i] = nu(Greville point of dof i) per
    velocity component; D_Q[i] = 1/nu(Greville point of pressure dof i)."""
    dv = np.concatenate([_grid_eval(nu, c.grev) for c in disc.comps])
    dq = 1.0 / _grid_eval(nu, disc.grev_q)
    return dv, dq
