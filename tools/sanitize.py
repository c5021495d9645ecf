"""Small resident FAST run for compute-sanitizer (memcheck / racecheck / synccheck): device IC,
two device steps, two pipelined end-to-end steps, a FAST sweep through the C ABI.
  compute-sanitizer --tool racecheck python tools/sanitize.py
SAN_N / SAN_PPC / SAN_SEED choose the box (default 8192 / 256 / 3); with more work items than
resident warp slots (e.g. SAN_N=131072 SAN_PPC=64: 4096+ items against 148 x 20 slots) the
persistent sweeps reuse each warp's shared-memory tiles across items."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_16517_b200 as pkg  # noqa: E402

with pkg.Context(0, numerics=pkg.Numerics.Fast, layout=pkg.DeviceLayout.Resident) as ctx:
    n, ppc = int(os.environ.get("SAN_N", 8192)), int(os.environ.get("SAN_PPC", 256))
    store, grid, par = ctx.make_particles(n, ppc, int(os.environ.get("SAN_SEED", 3)))
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
