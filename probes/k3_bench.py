"""Time of the banded pressure solve kron_mass_apply (all modes; CUDA events, 10 repetitions after
3 warm-ups) on config 5's pressure block (516^3, p = 4) or N^3 for another n_el, under the K3
environment switches (FDP_K3_CHUNKS, FDP_K3_CHUNK_M1, FDP_K3_NO_CHUNK, FDP_K3_SMEM_KB,
FDP_K3_TILE_ALL, FDP_K3_SWEEP). usage: k3_bench.py [n_el] [p]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1712_00403_b200 as fdp
from oracle import univariate  # the probe only borrows the mass matrix builder
n_el = int(sys.argv[1]) if len(sys.argv) > 1 else 512
p = int(sys.argv[2]) if len(sys.argv) > 2 else 4
M = univariate.pressure_mass(p, n_el)
K = fdp.KronMass([M, M, M])
b = torch.randn(K.N, dtype=torch.float64, device="cuda"); x = torch.empty_like(b)
for _ in range(3):
    K.apply(b, x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(10):
    e0.record(); K.apply(b, x); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("FDP_"))
print(f"k3 n={M.shape[0]}^3 [{tag}] median {np.median(ts):.3f} ms min {min(ts):.3f} ms "
      f"({16 * 3 * K.N / np.median(ts) / 1e6:.0f} GB/s at 16 B/element/mode)", flush=True)
