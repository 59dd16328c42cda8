"""Key occupancy / scheduler / throughput lines of an ncu --page details csv."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[0]
iS, iM, iU, iV = (h.index(x) for x in ("Section Name", "Metric Name", "Metric Unit", "Metric Value"))
want = ("Duration", "Executed Ipc Active", "Issue Slots Busy", "Achieved Active Warps Per SM",
        "Theoretical Active Warps per SM", "Eligible Warps Per Scheduler", "Registers Per Thread",
        "Grid Size", "Block Size", "Waves Per SM", "L1/TEX Hit Rate", "L2 Hit Rate", "DRAM Throughput",
        "Dynamic Shared Memory Per Block", "Block Limit Registers", "Block Limit Shared Mem")
for r in rows[1:]:
    if r[iM] in want:
        print(f"{r[iM][:40]:40s} {r[iV]:>12s} {r[iU]}")
