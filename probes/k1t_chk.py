import os, sys, json
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_1712_00403_b200 as fdp, synth
w = synth.CONFIGS[5]
gd = fdp.discretization(w.dim, w.disc, w.p, w.n_el)
P = fdp.build_block(gd)
r = torch.randn(1, gd.n_total, dtype=torch.float64, device="cuda"); s = torch.empty_like(r)
ws = P.workspace(1)
if os.environ.get("K1T_DBG"):
    import ctypes
    fdp.lib.fdp_k1t_set_dbg.argtypes = [ctypes.c_int]
    fdp.lib.fdp_k1t_set_dbg(int(os.environ["K1T_DBG"]))
a0, b0 = fdp.lib.fdp_debug_k1_launches(1), fdp.lib.fdp_debug_k1_launches(0)
P.apply(r, s, batch=1, workspace=ws); torch.cuda.synchronize()
print("k1t launches", fdp.lib.fdp_debug_k1_launches(1) - a0, "k1f", fdp.lib.fdp_debug_k1_launches(0) - b0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
P.profile(True); P.apply(r, s, batch=1, workspace=ws); torch.cuda.synchronize()
P.apply(r, s, batch=1, workspace=ws); torch.cuda.synchronize()
prof = P.profile_read(); P.profile(False)
print("dbg", os.environ.get("K1T_DBG", "0"), "K1t launch ms", [round(p[1], 3) for p in prof if p[0] == 0])
