"""Replicates the host-buffer pipeline of config 2 with torch streams and times each piece with
events on its own stream (diagnostic for block_precond_apply_host)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_1712_00403_b200 as fdp
import synth

w = synth.CONFIGS[2]
gd = fdp.discretization(w.dim, w.disc, w.p, w.n_el)
P = fdp.build_block(gd)
n = gd.n_total
o = [0]
for sz in gd.sizes:
    o.append(o[-1] + sz)
rh = torch.from_numpy(fdp.host_empty((n,)))
sh = torch.from_numpy(fdp.host_empty((n,)))
rd = torch.empty(n, dtype=torch.float64, device="cuda")
sd = torch.empty(n, dtype=torch.float64, device="cuda")
cin, cout, comp = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
wss = [torch.empty(f.workspace_bytes(1) // 8 + 1, dtype=torch.float64, device="cuda") for f in P.fds]
units = [3, 0, 1, 2]
E = lambda: torch.cuda.Event(enable_timing=True)


def run():
    t0 = E()
    t0.record()
    cin.wait_event(t0)
    ev_in, marks = [], {}
    with torch.cuda.stream(cin):
        for u in units:
            rd[o[u]:o[u + 1]].copy_(rh[o[u]:o[u + 1]], non_blocking=True)
            e = E()
            e.record()
            ev_in.append(e)
    ev_done = []
    for u, e in zip(units, ev_in):
        comp.wait_event(e)
        with torch.cuda.stream(comp):
            s0 = E(); s0.record()
            if u == 3:
                P.mass.apply(rd[o[3]:o[4]], sd[o[3]:o[4]])
            else:
                P.fds[u].apply(rd[o[u]:o[u + 1]], sd[o[u]:o[u + 1]], workspace=wss[u])
            s1 = E(); s1.record()
            marks[u] = (s0, s1)
            ev_done.append(s1)
    outs = []
    for u, e in zip(units, ev_done):
        cout.wait_event(e)
        with torch.cuda.stream(cout):
            sh[o[u]:o[u + 1]].copy_(sd[o[u]:o[u + 1]], non_blocking=True)
            e2 = E(); e2.record()
            outs.append(e2)
    torch.cuda.synchronize()
    rel = lambda e: t0.elapsed_time(e) * 1e3
    return {"h2d_done": [round(rel(e), 1) for e in ev_in],
            "compute": {u: (round(rel(a), 1), round(rel(b), 1)) for u, (a, b) in marks.items()},
            "d2h_done": [round(rel(e), 1) for e in outs]}


for _ in range(3):
    r = run()
print(json.dumps(r))


# the same schedule captured in one CUDA graph (host out of the loop), timed over replays
def sched():
    t0 = torch.cuda.Event()
    t0.record()
    cin.wait_event(t0)
    cout.wait_event(t0)
    comp.wait_event(t0)
    ev_in = []
    with torch.cuda.stream(cin):
        for u in units:
            rd[o[u]:o[u + 1]].copy_(rh[o[u]:o[u + 1]], non_blocking=True)
            e = torch.cuda.Event()
            e.record()
            ev_in.append(e)
    ev_done = []
    for u, e in zip(units, ev_in):
        comp.wait_event(e)
        with torch.cuda.stream(comp):
            if u == 3:
                P.mass.apply(rd[o[3]:o[4]], sd[o[3]:o[4]])
            else:
                P.fds[u].apply(rd[o[u]:o[u + 1]], sd[o[u]:o[u + 1]], workspace=wss[u])
            e2 = torch.cuda.Event()
            e2.record()
            ev_done.append(e2)
    for u, e in zip(units, ev_done):
        cout.wait_event(e)
        with torch.cuda.stream(cout):
            sh[o[u]:o[u + 1]].copy_(sd[o[u]:o[u + 1]], non_blocking=True)
    cur = torch.cuda.current_stream()
    cur.wait_stream(cout)
    cur.wait_stream(cin)
    cur.wait_stream(comp)


g = torch.cuda.CUDAGraph()
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    sched()
torch.cuda.synchronize()
with torch.cuda.graph(g):
    sched()
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50):
    g.replay()
b.record()
torch.cuda.synchronize()
print(json.dumps({"graph_schedule_us": a.elapsed_time(b) / 50 * 1e3}))
