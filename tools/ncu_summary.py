"""Key metrics per kernel from an .ncu-rep (raw page)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
keys = ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "launch__occupancy_limit_registers", "launch__grid_size"]
stalls = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    name = r[hdr.index("Kernel Name")][:70]
    print("==", name)
    for k in keys:
        if k in hdr:
            print(f"   {k:70s} {r[hdr.index(k)]} {rows[1][hdr.index(k)]}")
    st = sorted(((float(r[hdr.index(k)] or 0), k) for k in stalls), reverse=True)[:7]
    print("   stalls/issue:", ", ".join(f"{k[34:-27]}={v:.2f}" for v, k in st))
