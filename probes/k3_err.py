"""Error of the banded pressure solve against the oracle's Kronecker inverse on a 516 x 64 x 128
block (p = 4, 3, 2): relative L2 and max-abs, under the current FDP_K3_* switches."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1712_00403_b200 as fdp
from oracle import mass as omass, univariate
Ms = [univariate.pressure_mass(4, 512), univariate.pressure_mass(3, 61), univariate.pressure_mass(2, 126)]
km = omass.KronMass(Ms); N = int(np.prod(km.dims))
b = np.random.default_rng(3).standard_normal(N)
x = fdp.KronMass(Ms).apply(torch.from_numpy(b).cuda()).cpu().numpy()
ref = km.inverse(b)
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("FDP_"))
print(f"k3 err [{tag}] dims {km.dims}: rel L2 {np.linalg.norm(x-ref)/np.linalg.norm(ref):.3e} max-abs {np.max(np.abs(x-ref))/np.max(np.abs(ref)):.3e}")
