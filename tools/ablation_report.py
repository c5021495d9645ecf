"""Summarise tools/layout_ablation.sh outputs into profiles/<tag>_layout_ablation.md."""
import csv, io, json, re, sys
from collections import defaultdict
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
rows = []
kern = {}
for L in ("aos", "convert", "resident"):
    d = json.loads(open(f"gpurun_out/abl_{L}.json").read().strip().splitlines()[-1])
    rows.append((L, d))
    txt = open(f"gpurun_out/abl_ncu_{L}.csv").read()
    txt = txt[txt.index('"ID"'):]
    agg = defaultdict(lambda: defaultdict(float))
    cnt = defaultdict(int)
    seen = set()
    for r in csv.DictReader(io.StringIO(txt)):
        name = r["Kernel Name"]
        m = re.search(r"(\w+_kernel)", name)
        k = m.group(1) if m else name
        if "10FastPolicy" in name or "FastPolicy" in name:
            k += "<Fast>"
        key = (r["ID"], k)
        if key not in seen:
            seen.add(key)
            cnt[k] += 1
        v = float(r["Metric Value"].replace(",", ""))
        u = r["Metric Unit"]
        scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e3, "msecond": 1e6}.get(u, 1.0)
        agg[k][r["Metric Name"]] += v * scale
    kern[L] = (agg, cnt)
n = rows[0][1]["config"]["n"]
with open(f"profiles/{tag}_layout_ablation.md", "w") as f:
    f.write(f"# Layout ablation (BASELINE config 4), n = {n}, ppc = 1024, FAST numerics\n\n")
    f.write("Produced by `tools/layout_ablation.sh` + `tools/ablation_report.py` on one B200. "
            "Step = kick1, drift, rebin, density, force, kick2 (device-resident, CUDA events). "
            "Per-kernel DRAM bytes from one ncu pass (`--clock-control none`).\n\n")
    f.write("| layout | ms/step | kick1 | drift | rebin | density | force | kick2 | pairs/s |\n|---|---|---|---|---|---|---|---|---|\n")
    for L, d in rows:
        p = d["phase_ms"]
        f.write(f"| {L} | {d['ms_per_step']:.2f} | {p['kick1']:.3f} | {p['drift']:.3f} | {p['rebin']:.3f} | "
                f"{p['density']:.2f} | {p['force']:.2f} | {p['kick2']:.3f} | {d['value']:.3e} |\n")
    f.write("\n## Per-kernel DRAM traffic per particle (bytes; algorithmic: drift 80, kick1 80, kick2 192)\n\n")
    f.write("| layout | kernel | launches | time us/launch | DRAM B/particle | FP64 pipe % |\n|---|---|---|---|---|---|\n")
    for L in ("aos", "convert", "resident"):
        agg, cnt = kern[L]
        for k in sorted(agg):
            c = max(cnt[k], 1)
            t = agg[k].get("gpu__time_duration.sum", 0) / c / 1e3
            dram = (agg[k].get("dram__bytes_read.sum", 0) + agg[k].get("dram__bytes_write.sum", 0)) / c / n
            fp = agg[k].get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0) / c
            f.write(f"| {L} | {k} | {cnt[k]} | {t:.1f} | {dram:.1f} | {fp:.1f} |\n")
print(open(f"profiles/{tag}_layout_ablation.md").read())
