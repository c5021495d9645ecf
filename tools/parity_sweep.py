"""Randomised parity sweep on the GPU (a wider net than tests/test_gpu_parity.py).

For seeded random configurations (n, ppc, IC kind, seed) the density and force sweeps run
through the C ABI with EXACT numerics (must be byte-identical to the oracle) and FAST numerics
(per field |gpu - ref| <= 1e-10 |ref| + 1e-10 rms(ref); density may flip the h-round count
for <= 0.1 % of particles), on the resident layout. Writes a markdown table.

    python tools/parity_sweep.py [--configs 24] [--seed 2026] [--out gpurun_out/parity_sweep.md]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2502_16517_b200 as pkg  # noqa: E402
from paper_2502_16517_b200 import DeviceLayout, KernelId, Numerics  # noqa: E402
from oracle import Oracle  # noqa: E402  (test-only checker)

FIELDS = {KernelId.Density: ["h", "rho", "wcount", "rho_dh", "rot_v", "div_v"],
          KernelId.Force: ["a", "u_dt", "v_sig", "h_dt"]}


def run(recs0, par, ppc, numerics, k):
    recs = recs0.copy()
    store = pkg.ParticleStore(recs, np.arange(len(recs), dtype=np.int64), pkg.Layout.Continuous)
    grid = pkg.build_grid(store, pkg.InitConfig(n=len(recs), ppc=ppc))
    with pkg.Context(0, numerics=numerics, layout=DeviceLayout.Resident) as ctx:
        ctx.bind(grid)
        ctx.run_sweep(k, par)
    return recs, grid


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, default=24)
    ap.add_argument("--seed", type=int, default=2026)
    ap.add_argument("--out", default="gpurun_out/parity_sweep.md")
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    orc = Oracle()
    rows, fails = [], 0
    for c in range(a.configs):
        ppc = int(rng.choice([16, 32, 64, 128, 256, 512, 1024, 2048]))
        n = int(rng.integers(max(60, 2 * ppc), 80000 if ppc < 2048 else 40000))
        kind = int(rng.random() < 0.3)
        seed = int(rng.integers(1, 1 << 30))
        t0 = time.time()
        recs0, par = orc.make_particles(n, ppc, seed, kind=kind)
        for k in (KernelId.Density, KernelId.Force):
            ref = recs0.copy()
            ex, grid = run(recs0, par, ppc, Numerics.Exact, k)
            orc.sweep(int(k), ref, grid.nx, grid.ny, grid.cell_size, grid.cell_begin,
                      grid.local_idx, par)
            exact_ok = ex.tobytes() == ref.tobytes()
            fa, _ = run(recs0, par, ppc, Numerics.Fast, k)
            ok = np.ones(n, bool)
            worst = 0.0
            for f in FIELDS[k]:
                g, r = fa[f].astype(np.float64), ref[f].astype(np.float64)
                scale = np.sqrt(np.mean(r * r))
                err = np.abs(g - r)
                ok &= (err <= 1e-10 * np.abs(r) + 1e-10 * scale).reshape(n, -1).all(axis=1)
                rel = err / (np.abs(r) + scale + 1e-300)
                worst = max(worst, float(rel.max()))
            # FAST sweeps leave every other record byte untouched
            other = all(fa[nm].tobytes() == ref[nm].tobytes() for nm in ref.dtype.names
                        if nm not in FIELDS[k] and nm != "flags")
            flips = int(np.count_nonzero(~ok))
            fast_ok = other and (flips <= max(1, n // 1000) if k == KernelId.Density else flips == 0)
            fails += (not exact_ok) + (not fast_ok)
            rows.append((c, n, ppc, "clustered" if kind else "uniform", seed, grid.nx, k.name,
                         "yes" if exact_ok else "NO", f"{worst:.2e}", flips,
                         "ok" if fast_ok else "FAIL", f"{time.time() - t0:.1f}"))
            print(rows[-1], flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as fh:
        fh.write(f"# Randomised parity sweep (tools/parity_sweep.py --seed {a.seed})\n\n")
        fh.write("EXACT: byte-identical to the oracle. FAST: worst |gpu-ref| / (|ref| + rms) over "
                 "the kernel's output fields; flips = particles outside 1e-10 (density: h-round "
                 "threshold flips, <= 0.1 % allowed).\n\n")
        fh.write("| # | n | ppc | IC | seed | nx | kernel | EXACT bitwise | FAST worst rel | "
                 "FAST flips | FAST | s |\n|---|---|---|---|---|---|---|---|---|---|---|---|\n")
        for r in rows:
            fh.write("| " + " | ".join(str(x) for x in r) + " |\n")
        fh.write(f"\n{len(rows)} sweeps, {fails} failures.\n")
    print(f"{len(rows)} sweeps, {fails} failures")
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
