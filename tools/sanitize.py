"""Small resident FAST run for compute-sanitizer (memcheck / racecheck / synccheck): device IC,
two device steps, two pipelined end-to-end steps, a FAST sweep through the C ABI.
  compute-sanitizer --tool racecheck python tools/sanitize.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_16517_b200 as pkg  # noqa: E402

with pkg.Context(0, numerics=pkg.Numerics.Fast, layout=pkg.DeviceLayout.Resident) as ctx:
    store, grid, par = ctx.make_particles(8192, 256, 3)
    par.dt = 1e-3
    for _ in range(2):
        ctx.step(par)
    ctx.host_register(store.recs)
    for _ in range(2):
        ctx.step_host(par)
    ctx.host_unregister(store.recs)
    ctx.run_sweep(pkg.KernelId.Density, par)
    ctx.run_sweep(pkg.KernelId.Force, par)
    print("sanitize run ok, launches", ctx.launch_count())
