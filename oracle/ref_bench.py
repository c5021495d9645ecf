"""CPU timing of the UNMODIFIED reference on the bench workload.

Used only by bench.py's cpu_baseline leg and its ``--impl reference`` arm (test/baseline
infrastructure; never on the product path). One reference "step" mirrors the GPU step:
kick1 -> drift -> build_grid -> density -> force -> kick2 through the reference's own
run_sweep / build_grid (oracle/_ref, compiled from /root/reference), every kernel on every
cell (``sample_pairs=None``, the default: a full step, ~30 s at 2^21 on 16 cores).

``sample_pairs=x`` restricts density and force to random cells holding ~x pairs
(run_sweep skips cells whose local list is empty, kernels.cpp:548) and scales by pair
count. That is only for quick looks: unsampled cells never get their h updated, so later
sampled steps take extra h-rounds and the estimate is biased high.
Times are wall clock around each call (KernelTimes sums per-thread CPU time,
kernels.cpp:526-531).
"""
from __future__ import annotations

import os
import time

import numpy as np

from .loader import RefLib


def stencil_pairs(cb: np.ndarray, nx: int, ny: int) -> np.ndarray:
    """nl_c * na_c per cell for the deduplicated wrapped 3x3 stencil (grid.cpp:161-182)."""
    nl = np.diff(cb)
    cells = np.arange(nx * ny)
    cy, cx = np.divmod(cells, nx)
    na = np.zeros(nx * ny, np.int64)
    for c in range(nx * ny):
        seen = []
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                k = ((cy[c] + dy) % ny) * nx + (cx[c] + dx) % nx
                if k not in seen:
                    seen.append(k)
        na[c] = nl[seen].sum()
    return nl * na


class ReferenceStepper:
    def __init__(self, recs: np.ndarray, ppc: int, par, threads: int | None = None,
                 sample_pairs: float | None = None, seed: int = 0):
        self.ref = RefLib()
        self.recs = recs
        self.ppc = ppc
        self.par = par
        self.threads = threads or os.cpu_count() or 1
        self.sample_pairs = sample_pairs
        self.rng = np.random.default_rng(seed)

    def step(self) -> dict:
        """One reference step on the host records (in place); returns timings (s)."""
        r, par, th = self.ref, self.par, self.threads
        g_lin = r.grid(self.recs, self.ppc)  # the step's incoming grid (built last step)
        t = {}
        t0 = time.perf_counter()
        g_lin.run_sweep(3, par, threads=th)  # kick1
        t["kick1"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        g_lin.run_sweep(2, par, threads=th)  # drift
        t["drift"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        g = r.grid(self.recs, self.ppc)  # build_grid (grid.cpp:145-184), single-threaded
        t["rebin"] = time.perf_counter() - t0
        cb, _ = g.local_csr()
        per_cell = stencil_pairs(cb, g.nx, g.ny)
        total = int(per_cell.sum())
        if self.sample_pairs is None or self.sample_pairs >= total:
            sample = total  # the full step: every cell
        else:
            mask = self.rng.random(g.nx * g.ny) < self.sample_pairs / max(total, 1)
            if not mask.any():
                mask[self.rng.integers(g.nx * g.ny)] = True
            sample = int(per_cell[mask].sum())
            g.keep_cells(mask.astype(np.uint8))
        t0 = time.perf_counter()
        g.run_sweep(0, par, threads=th)  # density (sampled cells)
        t_den = time.perf_counter() - t0
        t0 = time.perf_counter()
        g.run_sweep(1, par, threads=th)  # force (sampled cells)
        t_for = time.perf_counter() - t0
        scale = total / max(sample, 1)
        t["density"] = t_den * scale
        t["force"] = t_for * scale
        t0 = time.perf_counter()
        g_lin.run_sweep(4, par, threads=th)  # kick2 (every particle)
        t["kick2"] = time.perf_counter() - t0
        g.close()
        g_lin.close()
        t["step"] = sum(t[k] for k in ("kick1", "drift", "rebin", "density", "force", "kick2"))
        t["workload_pairs"] = 2 * total
        t["sample_fraction"] = sample / max(total, 1)
        t["measured_seconds"] = t["kick1"] + t["drift"] + t["rebin"] + t_den + t_for + t["kick2"]
        return t
