"""Host-side mirror of the reference SPH API, backed by the B200 C-ABI.

Mirrors, with the same names, argument meaning and error behaviour:

* ``ParticleStore`` / ``CellGrid`` / ``InitConfig``      (grid.hpp:17-47)
* ``make_particles(cfg, par)``                           (grid.hpp:53, grid.cpp:76-143)
* ``build_grid(store, cfg)``                             (grid.hpp:54, grid.cpp:145-184)
* ``run_sweep(k, grid, par, path, order, guard, threads)`` (kernels.hpp:45-46)
* ``update_count(grid)``, ``drift_one/kick1_one/kick2_one`` (kernels.hpp:49-54)

Records live in one numpy array of the 272-byte ``PARTICLE_DTYPE``; ``store.all[k]`` is
the record index of the k-th particle of ``ParticleStore::all``. ``run_sweep`` hands the
flattened local lists to ``sph_run_sweep`` (upload of the kernel's A_in, sweep on the
device, download of its A_out) — there is no CPU compute path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .particle import (PARTICLE_DTYPE, RECORD_SIZE, DeviceLayout, Guard, KernelId, KernelTimes,
                       Layout, Numerics, Order, Path, SphParams)


def _check(ctx_handle, rc: int, what: str) -> None:
    if rc != _lib.SPH_OK:
        lib = _lib.load()
        msg = lib.sph_last_error(ctx_handle) if ctx_handle else b"no context"
        raise _lib.SphError(f"{what} failed ({rc}): {msg.decode(errors='replace')}")


def _cpar(par: SphParams) -> _lib.SphParamsC:
    return _lib.SphParamsC(par.dt, par.gamma, par.cfl, par.grav, par.target_wcount)


@dataclass
class InitConfig:
    n: int = 1000
    ppc: int = 64
    seed: int = 42
    layout: Layout = Layout.Scattered


@dataclass
class ParticleStore:
    """Records + the ParticleStore::all order (record index of each particle)."""
    recs: np.ndarray
    all: np.ndarray
    layout: Layout = Layout.Continuous

    def size(self) -> int:
        return len(self.all)

    def snapshot(self) -> np.ndarray:
        """Values of all particles in ``all`` order (grid.cpp:58-63)."""
        return self.recs[self.all].copy()

    def restore(self, snap: np.ndarray) -> None:
        """Write values back, preserving storage positions (grid.cpp:65-67)."""
        self.recs[self.all] = snap


@dataclass
class CellGrid:
    """Uniform grid on [0,1)^2; local lists as CSR of record indices (grid.hpp:32-40).

    The active list of a cell is the reference's deduplicated wrapped 3x3 stencil
    (grid.cpp:159-182) and is implied by (nx, ny); ``active(c)`` materialises it."""
    nx: int
    ny: int
    cell_size: float
    cell_begin: np.ndarray          # int64[ncells + 1]
    local_idx: np.ndarray           # int64[n], record indices, cell-major
    store: ParticleStore
    all_rank: np.ndarray = field(default=None)  # rank in store.all of each local entry

    def cells(self) -> int:
        return self.nx * self.ny

    def mean_ppc(self) -> float:
        return float(self.cell_begin[-1]) / self.cells() if self.cells() else 0.0

    def local(self, c: int) -> np.ndarray:
        return self.local_idx[self.cell_begin[c]:self.cell_begin[c + 1]]

    def stencil(self, c: int) -> list[int]:
        cy, cx = divmod(c, self.nx)
        out: list[int] = []
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                ci = ((cy + dy) % self.ny) * self.nx + (cx + dx) % self.nx
                if ci not in out:
                    out.append(ci)
        return out

    def active(self, c: int) -> np.ndarray:
        return np.concatenate([self.local(k) for k in self.stencil(c)])

    def record_pointers(self) -> np.ndarray:
        """Particle* of every local entry (the flattened CellGrid::local)."""
        base = self.store.recs.ctypes.data
        return (base + self.local_idx * RECORD_SIZE).astype(np.uint64)


def grid_nx(n: int, ppc: int) -> int:
    """grid.cpp:23-26."""
    cell = np.sqrt(float(ppc) / float(max(n, 1)))
    return max(1, int(np.floor(1.0 / cell)))


def build_grid(store: ParticleStore, cfg: InitConfig) -> CellGrid:
    """build_grid (grid.cpp:145-184): cell = clamp(floor(x*nx)), lists in ``all`` order.

    Writes each record's ``cell`` like the reference (grid.cpp:156)."""
    nx = grid_nx(store.size(), cfg.ppc)
    ny = nx
    x = store.recs["x"][store.all]
    cx = np.clip(np.floor(x[:, 0] * nx).astype(np.int64), 0, nx - 1)
    cy = np.clip(np.floor(x[:, 1] * nx).astype(np.int64), 0, ny - 1)
    ci = cy * nx + cx
    store.recs["cell"][store.all] = ci
    order = np.argsort(ci, kind="stable")              # stable: keeps ``all`` order per cell
    cb = np.zeros(nx * ny + 1, np.int64)
    np.cumsum(np.bincount(ci, minlength=nx * ny), out=cb[1:])
    return CellGrid(nx, ny, 1.0 / nx, cb, store.all[order].astype(np.int64), store,
                    all_rank=order.astype(np.int64))


def update_count(grid: CellGrid) -> int:
    """kernels.cpp:874-878."""
    return int(grid.cell_begin[-1])


class Context:
    """One device context (CUDA stream + device mirror of one bound grid)."""

    def __init__(self, device: int = 0, numerics: Numerics = Numerics.Fast,
                 layout: DeviceLayout = DeviceLayout.FromPath):
        self.lib = _lib.load()
        h = C.c_void_p()
        rc = self.lib.sph_create(device, C.byref(h))
        if rc != _lib.SPH_OK:
            raise _lib.SphError(f"sph_create(device={device}) failed ({rc}): no usable CUDA device")
        self.h = h.value
        self.grid: CellGrid | None = None
        self._ptrs: np.ndarray | None = None
        self.set_numerics(numerics)
        self.set_layout(layout)

    # -- configuration --
    def set_numerics(self, numerics: Numerics) -> None:
        _check(self.h, self.lib.sph_set_numerics(self.h, int(numerics)), "sph_set_numerics")
        self.numerics = Numerics(numerics)

    def set_layout(self, layout: DeviceLayout) -> None:
        _check(self.h, self.lib.sph_set_layout(self.h, int(layout)), "sph_set_layout")
        self.layout = DeviceLayout(layout)

    # -- binding / transfers --
    def bind(self, grid: CellGrid) -> None:
        ptrs = grid.record_pointers()
        cb = np.ascontiguousarray(grid.cell_begin, np.int64)
        rank = None if grid.all_rank is None else np.ascontiguousarray(grid.all_rank, np.int64)
        rc = self.lib.sph_bind(self.h, ptrs.ctypes.data, cb.ctypes.data, grid.nx, grid.ny,
                               grid.cell_size, None if rank is None else rank.ctypes.data)
        _check(self.h, rc, "sph_bind")
        self.grid, self._ptrs, self._rank = grid, ptrs, rank

    def set_owned_cells(self, mask: np.ndarray | None) -> None:
        """Sweep only the cells with mask[c] != 0 (domain decomposition); None = all."""
        self._need()
        if mask is None:
            _check(self.h, self.lib.sph_set_owned_cells(self.h, None), "sph_set_owned_cells")
        else:
            m = np.ascontiguousarray(mask, np.uint8)
            _check(self.h, self.lib.sph_set_owned_cells(self.h, m.ctypes.data), "sph_set_owned_cells")

    def _need(self) -> None:
        if self.grid is None:
            raise _lib.SphError("context has no bound grid")

    def upload(self) -> None:
        self._need()
        _check(self.h, self.lib.sph_upload(self.h, self._ptrs.ctypes.data), "sph_upload")

    def download(self) -> None:
        self._need()
        _check(self.h, self.lib.sph_download(self.h, self._ptrs.ctypes.data), "sph_download")

    def download_all(self) -> None:
        self._need()
        _check(self.h, self.lib.sph_download_all(self.h, self._ptrs.ctypes.data), "sph_download_all")

    # -- compute --
    def sweep(self, k: KernelId, par: SphParams, path: Path = Path.AosBaseline,
              order: Order = Order.LocalActive, guard: Guard = Guard.Branch) -> KernelTimes:
        self._need()
        t = _lib.SphTimesC()
        cp = _cpar(par)
        _check(self.h, self.lib.sph_sweep(self.h, int(k), C.byref(cp), int(path), int(order),
                                          int(guard), C.byref(t)), "sph_sweep")
        return KernelTimes(t.prologue_ns, t.compute_ns, t.epilogue_ns)

    def run_sweep(self, k: KernelId, par: SphParams, path: Path = Path.AosBaseline,
                  order: Order = Order.LocalActive, guard: Guard = Guard.Branch) -> KernelTimes:
        self._need()
        t = _lib.SphTimesC()
        cp = _cpar(par)
        _check(self.h, self.lib.sph_run_sweep(self.h, int(k), self._ptrs.ctypes.data, C.byref(cp),
                                              int(path), int(order), int(guard), C.byref(t)),
               "sph_run_sweep")
        return KernelTimes(t.prologue_ns, t.compute_ns, t.epilogue_ns)

    def rebin(self) -> None:
        self._need()
        _check(self.h, self.lib.sph_rebin(self.h), "sph_rebin")

    def step(self, par: SphParams) -> np.ndarray:
        """kick1 -> drift -> rebin -> density -> force -> kick2 on the device; per-phase ms."""
        self._need()
        ms = np.zeros(6, np.float64)
        cp = _cpar(par)
        _check(self.h, self.lib.sph_step(self.h, C.byref(cp), ms.ctypes.data), "sph_step")
        return ms

    def step_host(self, par: SphParams) -> np.ndarray:
        """End-to-end step on the host records of the bound grid (H2D, step, D2H);
        returns device ms for [H2D, kick1, drift, rebin, density, force, kick2, D2H]."""
        self._need()
        ms = np.zeros(8, np.float64)
        cp = _cpar(par)
        _check(self.h, self.lib.sph_step_host(self.h, self._ptrs.ctypes.data, C.byref(cp),
                                              ms.ctypes.data), "sph_step_host")
        return ms

    def host_register(self, arr: np.ndarray) -> None:
        _check(self.h, self.lib.sph_host_register(self.h, arr.ctypes.data, arr.nbytes),
               "sph_host_register")

    def host_unregister(self, arr: np.ndarray) -> None:
        _check(self.h, self.lib.sph_host_unregister(self.h, arr.ctypes.data), "sph_host_unregister")

    def make_particles(self, n: int, ppc: int, seed: int,
                       kind: int = 0) -> tuple[ParticleStore, CellGrid, SphParams]:
        """The reference IC computed on the device and left bound (continuous store).
        kind 0 = reference uniform IC, 1 = clustered variable-ppc IC (BASELINE config 3)."""
        cp = _lib.SphParamsC()
        _check(self.h, self.lib.sph_make_particles_ex(self.h, n, ppc, seed, int(kind),
                                                      C.byref(cp)), "sph_make_particles_ex")
        n = max(n, 1)
        recs = np.zeros(n, PARTICLE_DTYPE)
        _check(self.h, self.lib.sph_read_records(self.h, recs.ctypes.data), "sph_read_records")
        store = ParticleStore(recs, np.arange(n, dtype=np.int64), Layout.Continuous)
        grid = build_grid(store, InitConfig(n=n, ppc=ppc, seed=seed, layout=Layout.Continuous))
        self.grid = grid
        self._ptrs = grid.record_pointers()
        return store, grid, SphParams(cp.dt, cp.gamma, cp.cfl, cp.grav, cp.target_wcount)

    def make_particles_device(self, n: int, ppc: int, seed: int, kind: int = 0) -> SphParams:
        """make_particles bound on the device only (no host copy of the records): the
        starting point of a decomposed run, which then drops the other ranks' columns."""
        cp = _lib.SphParamsC()
        _check(self.h, self.lib.sph_make_particles_ex(self.h, n, ppc, seed, int(kind),
                                                      C.byref(cp)), "sph_make_particles_ex")
        self.grid = "device"  # bound, no host store
        self._ptrs = None
        return SphParams(cp.dt, cp.gamma, cp.cfl, cp.grav, cp.target_wcount)

    # -- device-resident slab decomposition (sph_dd_*; pointers are device addresses) --
    def count(self) -> int:
        return int(self.lib.sph_count(self.h))

    def dd_count(self, col_mask: np.ndarray) -> int:
        m = np.ascontiguousarray(col_mask, np.uint8)
        out = C.c_int64()
        _check(self.h, self.lib.sph_dd_count(self.h, m.ctypes.data, C.byref(out)), "sph_dd_count")
        return out.value

    def dd_export(self, col_mask: np.ndarray, recs_ptr: int, ranks_ptr: int, cap: int) -> int:
        m = np.ascontiguousarray(col_mask, np.uint8)
        out = C.c_int64()
        _check(self.h, self.lib.sph_dd_export(self.h, m.ctypes.data, recs_ptr, ranks_ptr, cap,
                                              C.byref(out)), "sph_dd_export")
        return out.value

    def dd_remove(self, col_mask: np.ndarray) -> None:
        m = np.ascontiguousarray(col_mask, np.uint8)
        _check(self.h, self.lib.sph_dd_remove(self.h, m.ctypes.data), "sph_dd_remove")

    def dd_append(self, recs_ptr: int, ranks_ptr: int, count: int) -> None:
        _check(self.h, self.lib.sph_dd_append(self.h, recs_ptr, ranks_ptr, count), "sph_dd_append")

    def dd_export_rho(self, col_mask: np.ndarray, out_ptr: int, cap: int) -> int:
        m = np.ascontiguousarray(col_mask, np.uint8)
        out = C.c_int64()
        _check(self.h, self.lib.sph_dd_export_rho(self.h, m.ctypes.data, out_ptr, cap,
                                                  C.byref(out)), "sph_dd_export_rho")
        return out.value

    def dd_import_rho(self, col_mask: np.ndarray, in_ptr: int, count: int) -> None:
        m = np.ascontiguousarray(col_mask, np.uint8)
        _check(self.h, self.lib.sph_dd_import_rho(self.h, m.ctypes.data, in_ptr, count),
               "sph_dd_import_rho")

    def dd_export_halo(self, col_mask: np.ndarray, out_ptr: int, ranks_ptr: int, cap: int) -> int:
        """Halo payload (x, v_pred, m, p, c: 7 doubles per particle) + all-ranks of the
        particles in the selected columns, in slot order."""
        m = np.ascontiguousarray(col_mask, np.uint8)
        out = C.c_int64()
        _check(self.h, self.lib.sph_dd_export_halo(self.h, m.ctypes.data, out_ptr, ranks_ptr, cap,
                                                   C.byref(out)), "sph_dd_export_halo")
        return out.value

    def dd_append_halo(self, in_ptr: int, ranks_ptr: int, count: int) -> None:
        _check(self.h, self.lib.sph_dd_append_halo(self.h, in_ptr, ranks_ptr, count),
               "sph_dd_append_halo")

    def sweep_cells(self, k: KernelId, par: SphParams, cell_mask: np.ndarray) -> None:
        """Force sweep on the owned cells with cell_mask[c] set."""
        m = np.ascontiguousarray(cell_mask, np.uint8)
        cp = _lib.SphParamsC(par.dt, par.gamma, par.cfl, par.grav, par.target_wcount)
        _check(self.h, self.lib.sph_sweep_cells(self.h, int(k), C.byref(cp), m.ctypes.data),
               "sph_sweep_cells")

    def set_stream(self, stream_ptr: int | None) -> None:
        """Run this context's device work on a caller's cudaStream_t (None: its own)."""
        _check(self.h, self.lib.sph_set_stream(self.h, stream_ptr), "sph_set_stream")

    def cell_counts(self) -> np.ndarray:
        """Local particle count of every cell of the bound grid."""
        st = self.stats()
        out = np.zeros(max(st["ncells"], 1), np.int64)
        _check(self.h, self.lib.sph_cell_counts(self.h, out.ctypes.data), "sph_cell_counts")
        return out[: st["ncells"]]

    def read_records_all(self) -> np.ndarray:
        """Every record of the context in slot order (device-only contexts included)."""
        out = np.zeros(max(self.count(), 1), PARTICLE_DTYPE)
        _check(self.h, self.lib.sph_read_records(self.h, out.ctypes.data), "sph_read_records")
        return out[: self.count()]

    def read_records(self) -> np.ndarray:
        self._need()
        out = np.zeros(len(self._ptrs), PARTICLE_DTYPE)
        _check(self.h, self.lib.sph_read_records(self.h, out.ctypes.data), "sph_read_records")
        return out

    def stats(self) -> dict:
        s = _lib.SphStatsC()
        _check(self.h, self.lib.sph_get_stats(self.h, C.byref(s)), "sph_get_stats")
        out = {name: getattr(s, name) for name, _ in s._fields_ if name != "pad0"}
        out["density_round_ms"] = list(s.density_round_ms)
        return out

    def pair_fractions(self) -> tuple[float, float, float, float]:
        """Exact shares of the active pairs with q < 2.5, < 1.5, < 0.5 in the current state
        (reference arithmetic), and the active-pair count (sph_pair_fractions)."""
        out = (C.c_double * 4)()
        _check(self.h, self.lib.sph_pair_fractions(self.h, out), "sph_pair_fractions")
        return out[0], out[1], out[2], out[3]

    def fp64_peak_tflops(self) -> float:
        v = C.c_double()
        _check(self.h, self.lib.sph_fp64_peak(self.h, C.byref(v)), "sph_fp64_peak")
        return v.value

    def launch_count(self) -> int:
        return int(self.lib.sph_launch_count(self.h))

    def synchronize(self) -> None:
        _check(self.h, self.lib.sph_synchronize(self.h), "sph_synchronize")

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.sph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


_default: Context | None = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


def make_particles(cfg: InitConfig, par: SphParams, ctx: Context | None = None) -> ParticleStore:
    """make_particles (grid.cpp:76-143): deterministic IC; calibrates par.target_wcount.

    The density / EOS / force initialisation passes run on the device with EXACT numerics,
    so the records are byte-identical to the reference's."""
    ctx = ctx or default_context()
    store, _, p = ctx.make_particles(cfg.n, cfg.ppc, cfg.seed)
    par.dt, par.gamma, par.cfl, par.grav, par.target_wcount = p.dt, p.gamma, p.cfl, p.grav, p.target_wcount
    if cfg.layout == Layout.Scattered:
        # values are layout-independent (test_sph.cpp:138-149); store them by id
        ids = store.recs["id"]
        recs = np.empty_like(store.recs)
        recs[ids] = store.recs
        store = ParticleStore(recs, np.arange(len(recs), dtype=np.int64), Layout.Scattered)
    return store


def run_sweep(k: KernelId, grid: CellGrid, par: SphParams, path: Path = Path.AosBaseline,
              order: Order = Order.LocalActive, guard: Guard = Guard.Branch, threads: int = 1,
              ctx: Context | None = None) -> KernelTimes:
    """Drop-in for soaview::sph::run_sweep (kernels.hpp:45-46) on the B200.

    ``threads`` is accepted for signature parity; the device decides its own parallelism.
    Path selects the device layout (AosBaseline: AoS in place, SoaView: per-call AoS->SoA
    conversion) unless the context forces one."""
    ctx = ctx or default_context()
    if ctx.grid is not grid:
        ctx.bind(grid)
    return ctx.run_sweep(k, par, path, order, guard)


# Single-particle ops (kernels.hpp:52-54): the exact streaming kernel on the device over the
# given records (sph_apply_records), without touching the context's bound grid.
def _one(kernel: KernelId, rec: np.ndarray, par: SphParams, ctx: Context | None) -> None:
    """``rec``: a contiguous PARTICLE_DTYPE array (one record, e.g. ``recs[i:i+1]``, or
    several), updated in place."""
    ctx = ctx or default_context()
    arr = np.asarray(rec)
    if arr.dtype != PARTICLE_DTYPE or not arr.flags.c_contiguous or not arr.flags.writeable:
        raise ValueError("expected a contiguous, writeable PARTICLE_DTYPE array view")
    _check(ctx.h, ctx.lib.sph_apply_records(ctx.h, int(kernel), arr.ctypes.data, arr.size,
                                            C.byref(_cpar(par))), "sph_apply_records")


def drift_one(rec: np.ndarray, par: SphParams, ctx: Context | None = None) -> None:
    _one(KernelId.Drift, rec, par, ctx)


def kick1_one(rec: np.ndarray, par: SphParams, ctx: Context | None = None) -> None:
    _one(KernelId.Kick1, rec, par, ctx)


def kick2_one(rec: np.ndarray, par: SphParams, ctx: Context | None = None) -> None:
    _one(KernelId.Kick2, rec, par, ctx)
