"""K1t per-role clock64 breakdown per launch of one apply (diagnostic build libfdp_prof.so).
usage: FDP_LIB_PATH=paper_1712_00403_b200/libfdp_prof.so python probes/k1t_roles.py CONFIG"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1712_00403_b200 as fdp, synth
cid = int(sys.argv[1]); w = synth.CONFIGS[cid]
gd = fdp.discretization(w.dim, w.disc, w.p, w.n_el)
P = fdp.build_block(gd)
r = torch.randn(w.batch, gd.n_total, dtype=torch.float64, device="cuda"); s = torch.empty_like(r)
ws = P.workspace(w.batch)
P.apply(r, s, batch=w.batch, workspace=ws); torch.cuda.synchronize()
buf = np.zeros(128, dtype=np.uint64)
rd = fdp.lib.fdp_k1t_prof_read
rd.argtypes = [ctypes.c_void_p]
rd(buf.ctypes.data)
P.profile(True)  # per-launch events: launches issued one by one, in order
base = int(fdp.lib.fdp_debug_k1_launches(1))
P.apply(r, s, batch=w.batch, workspace=ws); torch.cuda.synchronize()
n = int(fdp.lib.fdp_debug_k1_launches(1)) - base
prof = [p for p in P.profile_read() if p[0] == 0]
rd(buf.ctypes.data)
B = buf.reshape(8, 16).astype(float)
names = ["c.wait_full", "c.wait_stage", "c.total", "s.wait_tile", "s.total", "p.wait_empty", "p.total", "tiles"]
for i in range(n):
    row = B[(base + i) % 8]
    cw = 8 * 148  # consumer warps
    tiles = row[7] / 148
    print(f"cfg {cid} K1t launch {i}: {prof[i][1] if i < len(prof) else float('nan'):.3f} ms, tiles/CTA {tiles:.1f}, per tile (clk):"
          f" consumer total {row[2]/cw/tiles:.0f} wait_full {row[0]/cw/tiles:.0f} wait_stagebuf {row[1]/cw/tiles:.0f} |"
          f" store total {row[4]/(3*148)/tiles:.0f} wait_tile {row[3]/(3*148)/tiles:.0f} |"
          f" producer wait_empty {row[5]/148/tiles:.0f} issuing {row[9]/148/tiles:.0f} | consumer wait on a tile's first stage {row[8]/cw/tiles:.0f}", flush=True)
