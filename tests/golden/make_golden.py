"""Generate the golden vectors in tests/golden/ from the UNMODIFIED reference.

Runs the reference SPH code compiled from /root/reference by oracle/Makefile
(oracle/_ref/libsoaview_ref.so) and stores its outputs as small fixtures, so parity can be
checked where /root/reference does not exist (the GPU box):

  ic_<n>_<ppc>_<seed>.npz : make_particles IC (grid.cpp:76-143, continuous layout, records in
                            store.all order) + SphParams, and the records after one reference
                            run_sweep of each kernel on that IC (kernels.cpp:861-872)
  steps_<...>.npz         : three leapfrog steps kick1/drift/build_grid/density/force/kick2
  spline.npz              : kernel_w / kernel_dw on a q grid (spline.hpp:12-41)

Usage: python tests/golden/make_golden.py   (needs /root/reference; writes next to itself)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

CASES = [(400, 64, 11), (256, 64, 9), (1200, 256, 3)]
STEP_CASE = (1500, 64, 5, 1e-2)


def main():
    if not oracle.ref_available():
        oracle.build(ref=True)
    ref = oracle.RefLib()
    for n, ppc, seed in CASES:
        recs, par = ref.make_particles(n, ppc, seed, layout=1)
        out = {"ic": recs.copy(), "par": par.as_array()}
        for k, name in enumerate(["density", "force", "drift", "kick1", "kick2"]):
            r = recs.copy()
            g = ref.grid(r, ppc)
            g.run_sweep(k, par)
            out[name] = r
            g.close()
        np.savez_compressed(os.path.join(HERE, f"ic_{n}_{ppc}_{seed}.npz"), **out)

    n, ppc, seed, dt = STEP_CASE
    recs, par = ref.make_particles(n, ppc, seed, layout=1)
    p = par.as_array()
    p[0] = dt
    r = recs.copy()
    for _ in range(3):
        for k in (3, 2):  # kick1, drift (any grid enumerates every particle once)
            g = ref.grid(r, ppc)
            g.run_sweep(k, p)
            g.close()
        g = ref.grid(r, ppc)  # build_grid after drift (writes cell, new lists)
        for k in (0, 1, 4):
            g.run_sweep(k, p)
        g.close()
    np.savez_compressed(os.path.join(HERE, f"steps_{n}_{ppc}_{seed}.npz"), ic=recs, par=p, out=r)

    q = np.linspace(0.0, 2.7, 2701)
    w = np.array([ref.kernel_w(v) for v in q])
    dw = np.array([ref.kernel_dw(v) for v in q])
    np.savez_compressed(os.path.join(HERE, "spline.npz"), q=q, w=w, dw=dw)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
