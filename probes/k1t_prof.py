"""K1t phase breakdown (diagnostic): loads a libfdp built with -DFDP_K1T_PROF (FDP_LIB=...),
runs one config apply and prints warp-summed cycles waiting for stage data, in the K loop and in
the epilogue, per K1t launch."""
import ctypes, os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1712_00403_b200 as fdp
import synth
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
w = synth.CONFIGS[cid]
gd = fdp.discretization(w.dim, w.disc, w.p, w.n_el)
P = fdp.build_block(gd)
batch = w.batch
r = torch.randn(batch, gd.n_total, dtype=torch.float64, device="cuda"); s = torch.empty_like(r)
ws = P.workspace(batch)
prof = fdp.lib.fdp_k1t_prof
prof.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 320)()
for _ in range(3):
    P.apply(r, s, batch=batch, workspace=ws)
torch.cuda.synchronize()
prof(buf, 1)
P.apply(r, s, batch=batch, workspace=ws)
torch.cuda.synchronize()
prof(buf, 1)
names = {0: "nonK fwd", 1: "nonK bwd", 2: "nonK fwd+Lambda", 3: "nonK bwd+scale", 4: "KMAJ fwd", 5: "KMAJ bwd", 6: "KMAJ fwd+Lambda", 7: "KMAJ bwd+scale"}
for i in range(8):
    wait, kl, epi, tiles = list(buf)[4 * i:4 * i + 4]
    if tiles == 0:
        continue
    w0, slack, ready, cnt = list(buf)[32 + 4 * i:32 + 4 * i + 4]
    print(json.dumps({"cfg": cid, "kind": names[i],
                      "issue_to_need_cyc": round(slack / max(cnt, 1)), "issue_to_ready_cyc": round(ready / max(cnt, 1)),
                      "warp_tiles": tiles, "wait_frac_of_kloop": round(wait / kl, 3),
                      "epi_frac": round(epi / (kl + epi), 3), "kloop_cyc": round(kl / tiles), "epi_cyc": round(epi / tiles)}))

b = list(buf)
for i in (0, 4):
    ww = b[64 + 32 * i:64 + 32 * i + 16]
    print(names[i], "per-warp wait (M cycles):", [round(x / 1e6) for x in ww])
print("named-barrier cycles (all kinds) as a fraction of all K-loop cycles:",
      round(b[32] / max(1, sum(b[4 * i + 1] for i in range(8))), 3))
