"""Per-instruction stall samples of one kernel from an `ncu --page source --csv --print-source sass`
dump: totals by stall reason and by opcode, then the hottest instructions in address order.
usage: ncu_loop.py src.csv [kernel-index] [min-samples]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
which = int(sys.argv[2]) if len(sys.argv) > 2 else 0
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0
starts = [i for i, r in enumerate(rows) if any('Warp Stall Sampling' in c for c in r)]
st = starts[which]; en = starts[which + 1] if which + 1 < len(starts) else len(rows)
hdr = rows[st]
data = [r for r in rows[st + 1:en] if len(r) >= len(hdr) - 2]
ia, isrc = hdr.index('Address'), hdr.index('Source')
iall = [i for i, h in enumerate(hdr) if h.startswith('Warp Stall Sampling (All')][0]
cols = [i for i, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]
def f(x):
    try: return float(x)
    except: return 0.0
tot = {}; byop = {}
for r in data:
    toks = r[isrc].split()
    op = (toks[1] if toks[0].startswith('@') else toks[0]).split('.')[0]
    for c in cols:
        tot[hdr[c]] = tot.get(hdr[c], 0) + f(r[c])
        byop.setdefault(op, {}).setdefault(hdr[c], 0); byop[op][hdr[c]] += f(r[c])
s = sum(tot.values())
print("samples", s)
print(", ".join(f"{k[6:]} {100*v/s:.1f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]))
for op, d in sorted(byop.items(), key=lambda x: -sum(x[1].values()))[:8]:
    t = sum(d.values())
    print(f"  {op:8s} {100*t/s:5.1f}%  " + ", ".join(f"{k[6:]} {100*v/t:.0f}%" for k, v in sorted(d.items(), key=lambda x: -x[1])[:4]))
if thr:
    base = int(data[0][ia], 16)
    for r in data:
        if f(r[iall]) >= thr:
            top = max(cols, key=lambda c: f(r[c]))
            print(f"{int(r[ia],16)-base:5x} {f(r[iall]):6.0f} {hdr[top][6:]:10s} {r[isrc][:80]}")
