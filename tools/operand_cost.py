"""Static FP64 operand-read cost of a kernel's SASS (tools/operand_probe.cu, r2): an FP64
instruction issues to the pipe in 2 cycles per warp if it reads at most two distinct 64-bit
registers that are not served by the operand reuse cache, else one more cycle per extra
register. Prints, per loop (backward-branch span), the FP64 count and the extra cycles.

usage: python tools/operand_cost.py LIB.so KERNEL_REGEX [--list]"""
import re
import subprocess
import sys

lib, kre = sys.argv[1], sys.argv[2]
listing = "--list" in sys.argv
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs, cur = {}, None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = []
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m and cur:
        funcs[cur].append((int(m.group(1), 16), m.group(2).strip()))


def operands(ins):
    m = re.match(r"(@!?U?P\w+\s+)?(\w+)\S*\s+(.*)", ins)
    if not m:
        return None, []
    return m.group(2), [o.strip().lstrip("-|").rstrip("|") for o in m.group(3).split(",")][1:]


def annotate(body):
    """(addr, text, cost) with cost None for non-FP64; a .reuse operand of instruction k is
    served from the reuse cache to instruction k+1 when it sits in the same slot there."""
    out, cached = [], {}
    for a, t in body:
        op, ops = operands(t)
        c = None
        if op in ("DFMA", "DMUL", "DADD"):
            regs = set()
            for slot, o in enumerate(ops):
                r = o.split(".")[0]
                if re.match(r"R\d+$", r) and cached.get(slot) != r:
                    regs.add(r)
            c = max(2, len(regs))
        cached = {slot: o.split(".")[0] for slot, o in enumerate(ops) if ".reuse" in o}
        out.append((a, t, c))
    return out


for name, ins in funcs.items():
    if not re.search(kre, name):
        continue
    print("==", name, len(ins), "instructions")
    # loops: backward branches
    for addr, txt in ins:
        m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d+,\s*)?(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", txt)
        if not m or not m.group(1):
            continue
        tgt = int(m.group(1), 16)
        if tgt >= addr:
            continue
        body = annotate([(a, t) for a, t in ins if tgt <= a <= addr])
        fp = [c for a, t, c in body if c is not None]
        if len(fp) < 8:
            continue
        print(f"  loop {tgt:05x}-{addr:05x}: {len(body)} instr, {len(fp)} FP64, pipe {2*len(fp)} "
              f"+ extra {sum(fp)-2*len(fp)} cycles, 3-reg {sum(1 for c in fp if c > 2)}")
        if listing:
            for a, t, c in body:
                print(f"    {a:05x} {'*' if c and c > 2 else ' '} {t}")
