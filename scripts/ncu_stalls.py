"""Summarise an ncu report: per kernel duration, DRAM %, IPC and top stall reasons."""
import csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
st = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
def g(r, name):
    try: return r[hdr.index(name)]
    except ValueError: return "?"
for r in rows[2:]:
    vals = sorted(((h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                    float(r[hdr.index(h)] or 0)) for h in st), key=lambda x: -x[1])[:4]
    dram = g(r, "dram__bytes_read.sum"), g(r, "dram__bytes_write.sum")
    print(f"{g(r,'Kernel Name')[:34]:34s} t={g(r,'gpu__time_duration.sum'):>9s} dram_rd={dram[0]} wr={dram[1]} "
          f"ipc={g(r,'sm__inst_executed.avg.per_cycle_active')} stalls={[(a, round(b, 1)) for a, b in vals]}")
