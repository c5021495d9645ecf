"""FAST determinism over a longer run at BASELINE config 2 (diagnostic): two fresh contexts,
N device steps each, per-step density rounds / updates / round-1 time, and the final bytes."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_16517_b200 as pkg
from paper_2502_16517_b200 import Numerics, DeviceLayout

steps = int(os.environ.get("STEPS", 10))
outs = []
for rep in range(2):
    with pkg.Context(0, numerics=Numerics.Fast, layout=DeviceLayout.Resident) as ctx:
        store, grid, par = ctx.make_particles(1 << 21, 1024, 42)
        par.dt = 1e-4
        rows = []
        for s in range(steps):
            ctx.step(par)
            st = ctx.stats()
            rows.append((st["density_rounds"], st["density_updates"], round(st["density_round_ms"][1], 3)))
        print("rep", rep, rows, flush=True)
        outs.append(ctx.read_records().tobytes())
print("identical:", outs[0] == outs[1])
