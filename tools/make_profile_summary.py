"""Summarise ncu captures (gpurun_out/*.ncu-rep + launch list) into profiles/.

usage: python tools/make_profile_summary.py TAG
writes profiles/ncu_summary.json (read by bench.py for roofline.traffic),
profiles/<TAG>_summary.md and profiles/<TAG>_launches.csv
"""
import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import defaultdict

TAG = sys.argv[1] if len(sys.argv) > 1 else "r1"
G = "gpurun_out"
OUT = "profiles"
os.makedirs(OUT, exist_ok=True)

METRICS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),  # ns -> ms
    "dram_bytes_read": ("dram__bytes_read.sum", 1.0),
    "dram_bytes_write": ("dram__bytes_write.sum", 1.0),
    "fp64_pipe_active_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "registers": ("launch__registers_per_thread", 1.0),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "inst_executed": ("smsp__inst_executed.sum", 1.0),
    "avg_threads_per_inst": ("smsp__thread_inst_executed_per_inst_executed.ratio", 1.0),
    "sm_clock_mhz": ("sm__cycles_elapsed.avg.per_second", 1e-6),
}
UNITS = {"gpu__time_duration.sum": {"ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9},
         "dram__bytes_read.sum": {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9},
         "dram__bytes_write.sum": {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9},
         "sm__cycles_elapsed.avg.per_second": {"hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9,
                                              "cycle/second": 1, "cycle/nsecond": 1e9,
                                              "cycle/usecond": 1e6}}


def short(name):
    m = re.search(r"(\w+_kernel)<(?:sphb::)?(\w+)Policy", name)
    if m:
        return f"{m.group(1)}<{m.group(2)}Policy>"
    m = re.search(r"(\w+_kernel)", name)
    return m.group(1) if m else name[:60]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        d = {"name": short(r[hdr.index("Kernel Name")])}
        for k, (m, scale) in METRICS.items():
            if m not in hdr:
                continue
            v = float(r[hdr.index(m)] or 0)
            u = units[hdr.index(m)]
            if m in UNITS:
                v *= UNITS[m].get(u, 1.0)
                scale = {"gpu__time_duration.sum": 1e-6, "sm__cycles_elapsed.avg.per_second": 1e-6}.get(m, 1.0)
            d[k] = v * scale
        stalls = {h[34:-23]: float(r[hdr.index(h)] or 0) for h in hdr
                  if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")}
        d["top_stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:5])
        res.append(d)
    return res


summary = {"source": f"ncu --set full --clock-control none, tag {TAG} (tools/profile.sh)",
           "kernels": {}}
for rep in ("force", "density", "linear"):
    p = f"{G}/{rep}_{TAG}.ncu-rep"
    if not os.path.exists(p):
        continue
    for d in raw(p):
        summary["kernels"].setdefault(d["name"], d)
with open(f"{OUT}/ncu_summary.json", "w") as f:
    json.dump(summary, f, indent=1)

# launch list: per-kernel totals over the whole bench run (cold-cache, serialised)
lp = f"{G}/launches_{TAG}.csv"
tot = defaultdict(lambda: [0, 0.0])
rows_out = []
if os.path.exists(lp):
    txt = open(lp).read()
    txt = txt[txt.index('"ID"'):] if '"ID"' in txt else txt
    for r in csv.DictReader(io.StringIO(txt)):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        u = r.get("Metric Unit", "ns")
        ns = v * {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "nsecond": 1}.get(u, 1)
        k = short(r["Kernel Name"])
        tot[k][0] += 1
        tot[k][1] += ns
        rows_out.append((r["ID"], k, f"{ns / 1e3:.3f}"))
    with open(f"{OUT}/{TAG}_launches.csv", "w") as f:
        f.write("id,kernel,duration_us\n")
        for row in rows_out:
            f.write(",".join(row) + "\n")

with open(f"{OUT}/{TAG}_summary.md", "w") as f:
    f.write(f"# ncu summary ({TAG})\n\nCaptured with `tools/profile.sh {TAG}` on one B200 "
            "(`--clock-control none`); full reports are `gpurun_out/*_{TAG}.ncu-rep` (not tracked).\n\n")
    f.write("## Per-kernel (one launch each, --set full)\n\n")
    f.write("| kernel | ms | FP64 pipe % | issue % | warps % | regs | DRAM R+W MB | avg thr/inst | top stalls/issue |\n")
    f.write("|---|---|---|---|---|---|---|---|---|\n")
    for k, d in summary["kernels"].items():
        st = ", ".join(f"{a}={b:.2f}" for a, b in d["top_stalls_per_issue"].items())
        f.write(f"| {k} | {d.get('duration_ms', 0):.3f} | {d.get('fp64_pipe_active_pct', 0):.1f} | "
                f"{d.get('issue_active_pct', 0):.1f} | {d.get('warps_active_pct', 0):.1f} | "
                f"{d.get('registers', 0):.0f} | "
                f"{(d.get('dram_bytes_read', 0) + d.get('dram_bytes_write', 0)) / 1e6:.1f} | "
                f"{d.get('avg_threads_per_inst', 0):.1f} | {st} |\n")
    if tot:
        f.write("\n## Launch list totals (whole `bench.py --steps 2 --warmup 1 --e2e-steps 1` run, "
                "cold-cache serialised; compare shares, not absolutes)\n\n")
        f.write("| kernel | launches | total ms | share % |\n|---|---|---|---|\n")
        grand = sum(v[1] for v in tot.values())
        for k, (c, ns) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
            f.write(f"| {k} | {c} | {ns / 1e6:.3f} | {100 * ns / grand:.2f} |\n")
print(open(f"{OUT}/{TAG}_summary.md").read())
