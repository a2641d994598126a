import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
for i, r in enumerate(rows):
    if any('Warp Stall Sampling' in c for c in r):
        hdr = r; start = i + 1; break
print([h for h in hdr][:12])
idx_s = [i for i, h in enumerate(hdr) if h.startswith('Warp Stall Sampling (All')][0]
idx_src = [i for i, h in enumerate(hdr) if h in ('Source',)][0]
data = []
for r in rows[start:]:
    if len(r) <= idx_s: continue
    try: v = float(r[idx_s].replace(',', ''))
    except: continue
    data.append((v, r[idx_src][:110], r[0]))
tot = sum(d[0] for d in data)
data.sort(reverse=True)
for v, src, a in data[:40]:
    print(f"{100*v/tot:5.1f}%  {a:>6} {src}")
