"""Summarise an ncu SASS source page: per-instruction executed counts and stall samples.
usage: python tools/sass_hot.py REP KERNEL_REGEX [min_exec_fraction]"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
frac = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kre}", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr) and r[ix["Instructions Executed"]].isdigit()]
mx = max(int(r[ix["Instructions Executed"]] or 0) for r in data)
tot = sum(int(r[ix["Instructions Executed"]] or 0) for r in data)
samp = sum(int(r[ix["# Samples"]] or 0) for r in data)
print(rows[0][1], f"total warp-inst {tot:.3e}  samples {samp}")
from collections import Counter
ops = Counter()
for r in data:
    ex = int(r[ix["Instructions Executed"]] or 0)
    op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if op.startswith("@"):
        op = r[ix["Source"]].split()[1]
    ops[op.split(".")[0]] += ex
    if ex >= frac * mx:
        stalls = {k[6:]: int(r[ix[k]] or 0) for k in hdr if k.startswith("stall_") and "Not Issued" not in k}
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
        print(f"{r[ix['Address']][-5:]} {ex:>12} {float(r[ix['Avg. Threads Executed']] or 0):5.1f} "
              f"s={int(r[ix['# Samples']] or 0):5d} {r[ix['Source']].strip()[:60]:60s} {top}")
print("opcode mix (warp-inst):", [(k, f"{v/tot:.3f}") for k, v in ops.most_common(25)])
cls = Counter()
for r in data:
    ex = int(r[ix["Instructions Executed"]] or 0)
    toks = r[ix["Source"]].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    base = op.split(".")[0]
    if base in ("DADD", "DMUL", "DFMA", "DSETP", "DMNMX", "DSEL"):
        c = "fp64"
    elif base == "MUFU":
        c = "mufu"
    elif base in ("LDS", "STS", "LDG", "STG", "LDC", "LDSM", "ATOMS", "ATOMG", "RED"):
        c = "mem"
    elif base in ("BRA", "BSSY", "BSYNC", "EXIT", "BAR", "WARPSYNC", "CALL", "RET", "BREAK", "NOP"):
        c = "ctrl"
    else:
        c = "alu/other"
    cls[c] += ex
print("class mix:", {k: f"{v/tot:.3f}" for k, v in cls.most_common()}, f"total {tot:.3e}")
