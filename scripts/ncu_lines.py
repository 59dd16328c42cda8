"""Top CUDA source lines of an ncu 'source' page (--print-source cuda,sass csv) by stall samples."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
iW, iE = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
recs = []
for r in rows[hi + 1:]:
    if len(r) < len(h) or r[2] not in ("-", ""):
        continue
    try:
        recs.append((int(r[iE] or 0), int(r[iW] or 0), r[0], r[1][:100]))
    except ValueError:
        pass
te = sum(x[0] for x in recs) or 1
ts = sum(x[1] for x in recs) or 1
print("warp-instr", te, "stall samples", ts)
for e, w, l, s in sorted(recs, key=lambda x: -x[1])[:n]:
    print(f"{l:>5} inst {100 * e / te:5.1f}% stall {100 * w / ts:5.1f}%  {s}")
