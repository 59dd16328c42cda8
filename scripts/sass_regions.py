"""Per-region (split at barriers) instruction / stall-sample shares of an ncu --page source --csv --print-source sass dump."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
iS, iW, iE = h.index('Source'), h.index('Warp Stall Sampling (All Samples)'), h.index('Instructions Executed')
data = [(int(float(r[iE] or 0)), float(r[iW] or 0), r[iS].strip()) for r in rows[2:]]
warps = data[0][0]
T = sum(d[0] for d in data); S = sum(d[1] for d in data)
reg, cur = [], [0, 0, None, collections.Counter()]
for n, (e, w, s) in enumerate(data):
    if cur[2] is None: cur[2] = n
    cur[0] += e; cur[1] += w
    op = s.split()[1] if s.startswith('@') else (s.split() or [''])[0]
    cur[3][op.split('.')[0]] += e
    if 'BAR' in s or 'EXIT' in s:
        reg.append((cur[2], n, cur[0], cur[1], cur[3])); cur = [0, 0, None, collections.Counter()]
print(f"warps {warps} total inst/warp {T / warps:.0f}")
for a, b, e, w, c in reg:
    if e / T < 0.005: continue
    top = ', '.join(f"{k} {v / warps:.0f}" for k, v in c.most_common(6))
    print(f"lines {a}-{b}: inst {e / T * 100:5.1f}% samples {w / S * 100:5.1f}% per-warp {e / warps:.0f}  [{top}]")
