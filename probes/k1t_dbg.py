import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1712_00403_b200 as fdp
from oracle import fd as ofd
def rps(n, rng, shift):
    A = rng.standard_normal((n, n)); A = A @ A.T + shift * n * np.eye(n); return 0.5 * (A + A[::-1, ::-1])
case = eval(sys.argv[1]); batch = int(sys.argv[2])
rng = np.random.default_rng(1)
Ks = [rps(n, rng, 1.0) for n in case]; Ms = [rps(n, rng, 2.0) for n in case]
N = int(np.prod(case)); b = rng.standard_normal((batch, N))
x = fdp.FD(Ks, Ms, [2.0] + [1.0] * (len(case) - 1)).apply(torch.from_numpy(b).cuda(), batch=batch).cpu().numpy()
ref = ofd.FDSolver(Ks, Ms, [2.0] + [1.0] * (len(case) - 1))
print(case, batch, "err", max(np.linalg.norm(x[i] - ref.apply(b[i])) / np.linalg.norm(ref.apply(b[i])) for i in range(batch)), flush=True)
