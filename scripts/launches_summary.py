"""Per-kernel average device time and DRAM bytes from an ncu --csv launch list."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv")))
hdr = None
data = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        k = d["Kernel Name"].split("(")[0][-40:]
        data.setdefault(k, collections.defaultdict(list))[d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")))
tot = 0
for k, v in data.items():
    t = v["gpu__time_duration.sum"]
    n = len(t)
    avg = sum(t) / n / 1e3
    tot += avg
    print(f"{k:42s} n={n:3d} t={avg:8.1f}us rd={sum(v['dram__bytes_read.sum'])/n/1e6:7.1f}MB wr={sum(v['dram__bytes_write.sum'])/n/1e6:7.1f}MB")
print(f"sum of per-kernel averages: {tot:.1f} us")
