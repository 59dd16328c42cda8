"""Summarise an ncu SASS source page (csv): instruction mix and hot address ranges."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
iS, iE, iW = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
tot = 0; ops = collections.Counter(); stall = collections.Counter()
recs = []
for r in rows[2:]:
    if len(r) < len(h) or not (r[iE] or "0").isdigit(): continue
    n = int(r[iE] or 0); s = int(r[iW] or 0)
    op = r[iS].split()[0] if r[iS].split() else ""
    if op.startswith("@"): op = r[iS].split()[1]
    op = op.split(".")[0]
    ops[op] += n; stall[op] += s; tot += n
    recs.append((r[0], n, s, r[iS]))
print("total warp-instr", tot)
for op, n in ops.most_common(25):
    print(f"{op:10s} {n/1e6:9.2f}M {100*n/tot:5.1f}%  stall-samples {stall[op]}")
if len(sys.argv) > 2:
    thr = float(sys.argv[2])
    for a, n, s, src in recs:
        if n >= thr: print(a, n, s, src)
