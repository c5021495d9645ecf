"""ctypes loaders for the oracle libraries (TEST INFRASTRUCTURE).

* ``Oracle``  — liboracle.so, our C restatement of the reference path (sph_oracle.c).
* ``RefLib``  — _ref/libsoaview_ref.so, the unmodified reference sources compiled by
  oracle/Makefile plus the ref_capi.cpp wrapper.

Both operate on numpy arrays of ``PARTICLE_DTYPE`` records.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2502_16517_b200.particle import PARTICLE_DTYPE, SphParams

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsoaview_ref.so")

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_recp = np.ctypeslib.ndpointer(PARTICLE_DTYPE, flags="C_CONTIGUOUS")


def build(ref: bool = True) -> None:
    """Build liboracle.so (always) and _ref (when /root/reference is present)."""
    targets = ["oracle"]
    if ref and os.path.isdir("/root/reference/proj"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def oracle_available() -> bool:
    return os.path.exists(ORACLE_SO)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _par(par) -> np.ndarray:
    if isinstance(par, SphParams):
        return par.as_array()
    return np.ascontiguousarray(par, dtype=np.float64)


class Oracle:
    """Our plain-C restatement of the reference SPH path."""

    def __init__(self, path: str = ORACLE_SO):
        lib = C.CDLL(path)
        lib.orc_kernel_w.restype = C.c_double
        lib.orc_kernel_w.argtypes = [C.c_double]
        lib.orc_kernel_dw.restype = C.c_double
        lib.orc_kernel_dw.argtypes = [C.c_double]
        lib.orc_grid_nx.restype = C.c_int
        lib.orc_grid_nx.argtypes = [C.c_int64, C.c_int]
        lib.orc_build_grid.argtypes = [_recp, C.c_int64, C.c_int, C.c_int, _i64p, _i64p]
        lib.orc_sweep.restype = C.c_int
        lib.orc_sweep.argtypes = [C.c_int, _recp, C.c_int, C.c_int, C.c_double, _i64p, _i64p,
                                  _f64p, C.c_int, C.c_void_p]
        lib.orc_sweep_masked.restype = C.c_int
        lib.orc_sweep_masked.argtypes = [C.c_int, _recp, C.c_int, C.c_int, C.c_double, _i64p,
                                         _i64p, _f64p, C.c_int, C.c_void_p, C.c_void_p]
        lib.orc_mean_wcount.restype = C.c_double
        lib.orc_mean_wcount.argtypes = [_recp, C.c_int, C.c_int, _i64p, _i64p, C.c_int]
        lib.orc_make_proto.argtypes = [C.c_int64, C.c_int, C.c_uint64, _recp]
        lib.orc_make_particles_kind.restype = C.c_int
        lib.orc_make_particles_kind.argtypes = [C.c_int64, C.c_int, C.c_uint64, C.c_int, _recp,
                                                _f64p, C.c_int]
        lib.orc_make_particles.restype = C.c_int
        lib.orc_make_particles.argtypes = [C.c_int64, C.c_int, C.c_uint64, _recp, _f64p, C.c_int]
        lib.orc_pair_stats.argtypes = [_recp, C.c_int, C.c_int, _i64p, _i64p, C.c_void_p, C.c_int,
                                       _i64p]
        lib.orc_pair_stats_cell.argtypes = [_recp, C.c_int, C.c_int, _i64p, _i64p, C.c_int,
                                            C.c_int64, C.c_int, _i64p]
        for name in ("orc_drift_one", "orc_kick1_one", "orc_kick2_one"):
            getattr(lib, name).argtypes = [C.c_void_p, _f64p]
        self.lib = lib
        self.threads = os.cpu_count() or 1

    def kernel_w(self, q: float) -> float:
        return self.lib.orc_kernel_w(q)

    def kernel_dw(self, q: float) -> float:
        return self.lib.orc_kernel_dw(q)

    def grid_nx(self, n: int, ppc: int) -> int:
        return self.lib.orc_grid_nx(n, ppc)

    def build_grid(self, recs: np.ndarray, nx: int, ny: int | None = None):
        ny = nx if ny is None else ny
        cb = np.zeros(nx * ny + 1, np.int64)
        li = np.zeros(len(recs), np.int64)
        self.lib.orc_build_grid(recs, len(recs), nx, ny, cb, li)
        return cb, li

    def sweep(self, kernel: int, recs, nx, ny, cell_size, cb, li, par, threads=None,
              rounds: np.ndarray | None = None) -> None:
        rp = rounds.ctypes.data_as(C.c_void_p) if rounds is not None else None
        self.lib.orc_sweep(int(kernel), recs, nx, ny, cell_size, cb, li, _par(par),
                           threads or self.threads, rp)

    def sweep_masked(self, kernel: int, recs, nx, ny, cell_size, cb, li, par, cell_mask,
                     threads=None) -> None:
        m = np.ascontiguousarray(cell_mask, np.uint8)
        self.lib.orc_sweep_masked(int(kernel), recs, nx, ny, cell_size, cb, li, _par(par),
                                  threads or self.threads, None, m.ctypes.data)

    def mean_wcount(self, recs, nx, ny, cb, li, threads=None) -> float:
        return self.lib.orc_mean_wcount(recs, nx, ny, cb, li, threads or self.threads)

    def make_proto(self, n: int, ppc: int, seed: int) -> np.ndarray:
        out = np.zeros(max(n, 1), PARTICLE_DTYPE)
        self.lib.orc_make_proto(n, ppc, seed, out)
        return out

    def make_particles(self, n: int, ppc: int, seed: int, threads=None, kind: int = 0):
        """Continuous-layout IC: records sorted by (cell, id) + calibrated SphParams.
        kind 0 = reference uniform IC, 1 = clustered (variable ppc, BASELINE config 3)."""
        out = np.zeros(max(n, 1), PARTICLE_DTYPE)
        par = np.zeros(5, np.float64)
        self.lib.orc_make_particles_kind(n, ppc, seed, kind, out, par, threads or self.threads)
        return out, SphParams.from_array(par)

    def pair_stats(self, recs, nx, ny, cb, li, threads=None, cell_mask=None) -> np.ndarray:
        """[active pairs, r2>0, q<2.5, q<1.5, q<0.5] over the (masked) cells."""
        out = np.zeros(5, np.int64)
        m = None if cell_mask is None else np.ascontiguousarray(cell_mask, np.uint8)
        self.lib.orc_pair_stats(recs, nx, ny, cb, li, None if m is None else m.ctypes.data,
                                threads or self.threads, out)
        return out

    def pair_stats_cell(self, recs, nx, ny, cb, li, cell, i_stride=1, threads=None) -> np.ndarray:
        """pair_stats of one cell over every i_stride-th local (threads split the locals)."""
        out = np.zeros(5, np.int64)
        self.lib.orc_pair_stats_cell(recs, nx, ny, cb, li, int(cell), int(i_stride),
                                     threads or self.threads, out)
        return out

    def one(self, which: str, rec: np.ndarray, par) -> None:
        """drift_one / kick1_one / kick2_one on a single record (in place)."""
        getattr(self.lib, f"orc_{which}_one")(rec.ctypes.data_as(C.c_void_p), _par(par))


class RefGrid:
    def __init__(self, lib: "RefLib", handle, recs: np.ndarray):
        self.lib, self.h, self.recs = lib, handle, recs
        nx, ny, cs, at = C.c_int(), C.c_int(), C.c_double(), C.c_int64()
        lib.lib.ref_grid_info(handle, C.byref(nx), C.byref(ny), C.byref(cs), C.byref(at))
        self.nx, self.ny, self.cell_size, self.active_total = nx.value, ny.value, cs.value, at.value

    @property
    def cells(self) -> int:
        return self.nx * self.ny

    def local_csr(self):
        cb = np.zeros(self.cells + 1, np.int64)
        li = np.zeros(len(self.recs), np.int64)
        self.lib.lib.ref_grid_local_csr(self.h, self.recs.ctypes.data_as(C.c_void_p), cb, li)
        return cb, li

    def active_csr(self):
        cb = np.zeros(self.cells + 1, np.int64)
        ai = np.zeros(max(self.active_total, 1), np.int64)
        self.lib.lib.ref_grid_active_csr(self.h, self.recs.ctypes.data_as(C.c_void_p), cb, ai)
        return cb, ai[: self.active_total]

    def keep_cells(self, mask: np.ndarray) -> None:
        m = np.ascontiguousarray(mask, dtype=np.uint8)
        self.lib.lib.ref_grid_keep_cells(self.h, m.ctypes.data_as(C.c_void_p))

    def update_count(self) -> int:
        return self.lib.lib.ref_update_count(self.h)

    def run_sweep(self, kernel, par, path=0, order=0, guard=0, threads=1) -> np.ndarray:
        """reference run_sweep; returns [prologue, compute, epilogue, wall] ns."""
        t = np.zeros(4, np.int64)
        self.lib.lib.ref_run_sweep(self.h, int(kernel), _par(par), int(path), int(order),
                                   int(guard), int(threads), t)
        return t

    def close(self) -> None:
        if self.h:
            self.lib.lib.ref_grid_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class RefLib:
    """The unmodified reference implementation (oracle/_ref/libsoaview_ref.so)."""

    def __init__(self, path: str = REF_SO):
        lib = C.CDLL(path)
        lib.ref_record_size.restype = C.c_int
        lib.ref_kernel_w.restype = C.c_double
        lib.ref_kernel_w.argtypes = [C.c_double]
        lib.ref_kernel_dw.restype = C.c_double
        lib.ref_kernel_dw.argtypes = [C.c_double]
        lib.ref_make_particles.argtypes = [C.c_int64, C.c_int, C.c_uint64, C.c_int, C.c_void_p,
                                           _f64p]
        lib.ref_grid_create.restype = C.c_void_p
        lib.ref_grid_create.argtypes = [C.c_void_p, C.c_int64, C.c_int]
        lib.ref_grid_create_ordered.restype = C.c_void_p
        lib.ref_grid_create_ordered.argtypes = [C.c_void_p, C.c_int64, C.c_int, _i64p]
        lib.ref_grid_destroy.argtypes = [C.c_void_p]
        lib.ref_grid_info.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.ref_grid_local_csr.argtypes = [C.c_void_p, C.c_void_p, _i64p, _i64p]
        lib.ref_grid_active_csr.argtypes = [C.c_void_p, C.c_void_p, _i64p, _i64p]
        lib.ref_grid_keep_cells.argtypes = [C.c_void_p, C.c_void_p]
        lib.ref_update_count.restype = C.c_int64
        lib.ref_update_count.argtypes = [C.c_void_p]
        lib.ref_run_sweep.argtypes = [C.c_void_p, C.c_int, _f64p, C.c_int, C.c_int, C.c_int,
                                      C.c_int, _i64p]
        for name in ("ref_drift_one", "ref_kick1_one", "ref_kick2_one"):
            getattr(lib, name).argtypes = [C.c_void_p, _f64p]
        lib.ref_view_fields.restype = C.c_int
        lib.ref_view_fields.argtypes = [C.c_int, _i32p, C.c_int]
        self.lib = lib
        assert lib.ref_record_size() == PARTICLE_DTYPE.itemsize

    def kernel_w(self, q: float) -> float:
        return self.lib.ref_kernel_w(q)

    def kernel_dw(self, q: float) -> float:
        return self.lib.ref_kernel_dw(q)

    def make_particles(self, n: int, ppc: int, seed: int, layout: int = 1):
        """reference make_particles; records in store.all order + SphParams."""
        out = np.zeros(max(n, 1), PARTICLE_DTYPE)
        par = np.zeros(5, np.float64)
        self.lib.ref_make_particles(n, ppc, seed, layout, out.ctypes.data_as(C.c_void_p), par)
        return out, SphParams.from_array(par)

    def grid(self, recs: np.ndarray, ppc: int, order: np.ndarray | None = None) -> RefGrid:
        """reference build_grid with store.all = recs (or recs[order])."""
        assert recs.dtype == PARTICLE_DTYPE and recs.flags.c_contiguous
        if order is None:
            h = self.lib.ref_grid_create(recs.ctypes.data_as(C.c_void_p), len(recs), ppc)
        else:
            h = self.lib.ref_grid_create_ordered(recs.ctypes.data_as(C.c_void_p), len(recs), ppc,
                                                 np.ascontiguousarray(order, np.int64))
        return RefGrid(self, h, recs)

    def one(self, which: str, rec: np.ndarray, par) -> None:
        getattr(self.lib, f"ref_{which}_one")(rec.ctypes.data_as(C.c_void_p), _par(par))

    def view_fields(self, which: int):
        out = np.zeros(3 * 32, np.int32)
        k = self.lib.ref_view_fields(which, out, 32)
        return [tuple(out[3 * i: 3 * i + 3]) for i in range(k)]
