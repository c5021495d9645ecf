"""Which scheduling switch changes FAST step results, and by how much (diagnostic)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_16517_b200 as pkg
from paper_2502_16517_b200 import Numerics, DeviceLayout, KernelId

n, ppc, seed, kind = 131072, 64, 11, int(os.environ.get("KIND", 0))
def sweep_force(persist):
    os.environ["SPH_B200_F2_PERSIST"] = persist
    with pkg.Context(0, numerics=Numerics.Fast, layout=DeviceLayout.Resident) as ctx:
        store, grid, par = ctx.make_particles(n, ppc, seed, kind=kind)
        ctx.run_sweep(KernelId.Density, par)
        ctx.run_sweep(KernelId.Force, par)
        return ctx.read_records()
a = sweep_force("0"); b = sweep_force("1"); c = sweep_force("1")
print("persist vs persist identical:", b.tobytes() == c.tobytes())
d = np.abs(a["a"] - b["a"]).max(axis=1)
rel = d / (np.abs(a["a"]).max(axis=1) + 1e-300)
idx = np.nonzero(d)[0]
print("differing particles", len(idx), "max rel", rel.max(), "median rel of differing", np.median(rel[idx]) if len(idx) else 0)
print("first differing slots/cells:", idx[:10], a["cell"][idx[:10]])
for f in a.dtype.names:
    if a[f].tobytes() != b[f].tobytes():
        print("field differs:", f)
