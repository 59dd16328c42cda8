"""Per-kernel summary of an ncu --set full report -> JSON (committed under profiles/).

  python scripts/ncu_to_json.py gpurun_out/prof_C.ncu-rep profiles/r01_ncu_kernels.json
"""
import csv, json, subprocess, sys

rep, dst = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
keys = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_pct_peak": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "alu_pipe_pct_active": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct_active": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "lsu_shared_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "ipc": "sm__inst_executed.avg.per_cycle_active",
    "registers": "launch__registers_per_thread",
}
units = {r: u for r, u in zip(hdr, rows[1])}
out = {}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("unnamed>::", "")
    d = {}
    for k, m in keys.items():
        if m in hdr:
            v = r[hdr.index(m)].replace(",", "")
            try:
                v = float(v)
            except ValueError:
                continue
            u = units.get(m, "")
            if k == "duration_us" and u == "ns":
                v /= 1e3
            if k.startswith("dram_") and k.endswith("bytes"):
                v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            d[k] = v
    out.setdefault(name, []).append(d)
json.dump(out, open(dst, "w"), indent=1)
print(f"{len(out)} kernels -> {dst}")
