"""The reference's bench harness with the B200 path selectable.

Mirrors ``soaview::sph`` bench.hpp:11-64 / bench.cpp:93-233 — ``VariantSpec``,
``variant_string``, ``parse_variant``, ``BenchConfig``, ``BenchRecord``, ``run_bench``,
``to_csv`` — with the same variant grammar ("path,layout,order,guard" in any order), the
same record fields, the same CSV header and the same error behaviour (ppc <= 0 or
ppc > particles raise; reps == 0 returns no records). Sweeps run through
``Context.run_sweep`` (host records in, A_out back), so prologue / epilogue are the
host<->device copies of each kernel's view and compute is device time. Two extra variant
tokens pick the device numerics: ``exact`` (byte-identical to the CPU) and ``fast``.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .particle import Guard, KernelId, Layout, Numerics, Order, Path, SphParams
from .sph import CellGrid, Context, InitConfig, ParticleStore, build_grid, update_count

_PATH = {Path.AosBaseline: "aos-baseline", Path.SoaView: "soa-view"}
_LAYOUT = {Layout.Scattered: "scattered", Layout.Continuous: "continuous"}
_ORDER = {Order.LocalActive: "local-active", Order.ActiveLocal: "active-local"}
_GUARD = {Guard.Branch: "branch", Guard.Mask: "mask"}
_NUM = {Numerics.Fast: "fast", Numerics.Exact: "exact"}
KERNEL_NAMES = {KernelId.Density: "density", KernelId.Force: "force", KernelId.Drift: "drift",
                KernelId.Kick1: "kick1", KernelId.Kick2: "kick2"}  # kernels.cpp:726-739

CSV_HEADER = ("kernel,path,layout,order,guard,ppc,n,t_prologue_ns,t_compute_ns,t_epilogue_ns,"
              "t_total_ns,ns_per_update\n")  # bench.cpp:220-221


@dataclass
class VariantSpec:  # bench.hpp:11-16 (+ device numerics)
    path: Path = Path.AosBaseline
    layout: Layout = Layout.Scattered
    order: Order = Order.LocalActive
    guard: Guard = Guard.Branch
    numerics: Numerics = Numerics.Fast


def variant_string(v: VariantSpec) -> str:
    """bench.cpp:93-102 (numerics appended only when not the default)."""
    s = f"{_PATH[v.path]},{_LAYOUT[v.layout]},{_ORDER[v.order]},{_GUARD[v.guard]}"
    return s if v.numerics == Numerics.Fast else s + f",{_NUM[v.numerics]}"


def parse_variant(s: str) -> VariantSpec:
    """bench.cpp:104-133; raises ValueError("unknown variant token '...'") like `err`."""
    v = VariantSpec()
    table = {}
    for d, attr in ((_PATH, "path"), (_LAYOUT, "layout"), (_ORDER, "order"), (_GUARD, "guard"),
                    (_NUM, "numerics")):
        for k, tok in d.items():
            table[tok] = (attr, k)
    for tok in (t.strip() for t in s.split(",")):
        if tok not in table:
            raise ValueError(f"unknown variant token '{tok}'")
        setattr(v, table[tok][0], table[tok][1])
    return v


@dataclass
class BenchConfig:  # bench.hpp:23-32
    kernels: list = field(default_factory=list)
    variants: list = field(default_factory=list)
    ppcs: list = field(default_factory=lambda: [1024])
    particles: int = 100000
    reps: int = 5
    seed: int = 42
    threads: int = 1
    cross_check: bool = True  # compare against the exact device path (bitwise reference)


@dataclass
class KernelTimesRec:
    prologue_ns: int = 0
    compute_ns: int = 0
    epilogue_ns: int = 0

    def total(self) -> int:
        return self.prologue_ns + self.compute_ns + self.epilogue_ns


@dataclass
class BenchRecord:  # bench.hpp:34-54
    kernel: KernelId
    variant: VariantSpec
    ppc: int = 0
    n: int = 0
    t_prologue_ns: int = 0
    t_compute_ns: int = 0
    t_epilogue_ns: int = 0
    t_total_ns: int = 0
    ns_per_update: float = 0.0
    reps: list = field(default_factory=list)
    cross_max_rel: float = 0.0

    def conversion_share(self) -> float:
        return 0.0 if self.t_total_ns == 0 else (self.t_prologue_ns + self.t_epilogue_ns) / self.t_total_ns


_OUT_FIELDS = {  # cross_compare field lists, bench.cpp:32-82
    KernelId.Density: ["rho", "wcount", "rho_dh", "rot_v", "div_v", "h"],
    KernelId.Force: ["a", "u_dt", "v_sig", "h_dt"],
    KernelId.Drift: ["x", "u_pred"],
    KernelId.Kick1: ["v", "u", "dt_next"],
    KernelId.Kick2: ["v", "v_pred", "u", "u_pred", "c", "p", "dt_next", "h_dt"],
}


def _rel_diff(a, b):  # bench.cpp:24-28
    d = np.abs(a - b)
    den = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-30)
    return np.where(d == 0, 0.0, d / den)


def _median(v):
    return sorted(v)[len(v) // 2]  # bench.cpp:19-22


def run_bench(cfg: BenchConfig, ctx: Context | None = None) -> list[BenchRecord]:
    """bench.cpp:135-217 on the device: per ppc, one IC per store layout (the reference IC
    from sph_make_particles), one warm-up sweep, `reps` timed sweeps from the restored IC,
    medians; soa-view records are cross-checked against the exact device sweep. (The
    reference's cross_compare runs the CPU path; product code here may not call the
    test-only oracle, so this mirror compares with the EXACT device sweep, which the GPU
    tests pin byte for byte to the reference. The reference's own run_bench, cross-checking
    against its CPU rows, runs on the B200 through the link-time drop-in: INTEGRATION.md
    §2b, profiles/r2_reference_bench_harness_gpu.csv.)"""
    out: list[BenchRecord] = []
    if cfg.reps <= 0:
        return out
    own = ctx is None
    ctx = ctx or Context(0)
    try:
        for ppc in cfg.ppcs:
            if ppc <= 0:
                raise RuntimeError("cells-per-particle target must be positive")
            if ppc > cfg.particles:
                raise RuntimeError(f"ppc {ppc} exceeds the particle count {cfg.particles}")
            slots = {}

            def slot_for(lay):
                if lay not in slots:
                    store, _, par = ctx.make_particles(cfg.particles, ppc, cfg.seed)
                    if lay == Layout.Scattered:  # same values, storage by id (grid.cpp:103-116)
                        recs = np.empty_like(store.recs)
                        recs[store.recs["id"]] = store.recs
                        store = ParticleStore(recs, np.arange(len(recs), dtype=np.int64), lay)
                    grid = build_grid(store, InitConfig(n=cfg.particles, ppc=ppc, seed=cfg.seed,
                                                        layout=lay))
                    slots[lay] = (store, grid, par, store.snapshot())
                return slots[lay]

            refs = {}

            def ref_for(lay, k):
                key = (lay, k)
                if key not in refs:
                    store, grid, par, ic = slot_for(lay)
                    store.restore(ic)
                    ctx.set_numerics(Numerics.Exact)
                    ctx.bind(grid)
                    ctx.run_sweep(k, par)
                    refs[key] = store.snapshot()
                return refs[key]

            for k in cfg.kernels:
                for v in cfg.variants:
                    store, grid, par, ic = slot_for(v.layout)
                    rec = BenchRecord(kernel=k, variant=v, ppc=ppc, n=store.size())
                    ctx.set_numerics(v.numerics)
                    store.restore(ic)
                    ctx.bind(grid)
                    ctx.run_sweep(k, par, v.path, v.order, v.guard)  # warm-up
                    for r in range(cfg.reps):
                        store.restore(ic)
                        t = ctx.run_sweep(k, par, v.path, v.order, v.guard)
                        rec.reps.append(KernelTimesRec(t.prologue_ns, t.compute_ns, t.epilogue_ns))
                        if r == 0 and cfg.cross_check and v.path == Path.SoaView:
                            got = store.snapshot()
                            ref = ref_for(v.layout, k)
                            ctx.set_numerics(v.numerics)
                            ctx.bind(grid)
                            rec.cross_max_rel = max(float(_rel_diff(got[f], ref[f]).max())
                                                    for f in _OUT_FIELDS[k])
                    rec.t_prologue_ns = _median([t.prologue_ns for t in rec.reps])
                    rec.t_compute_ns = _median([t.compute_ns for t in rec.reps])
                    rec.t_epilogue_ns = _median([t.epilogue_ns for t in rec.reps])
                    rec.t_total_ns = _median([t.total() for t in rec.reps])
                    upd = update_count(grid)
                    rec.ns_per_update = rec.t_total_ns / upd if upd else 0.0
                    out.append(rec)
    finally:
        if own:
            ctx.close()
    return out


def to_csv(records: list[BenchRecord]) -> str:
    """bench.cpp:219-233 (same header and column formats)."""
    out = CSV_HEADER
    for r in records:
        v = r.variant
        out += (f"{KERNEL_NAMES[r.kernel]},{_PATH[v.path]},{_LAYOUT[v.layout]},{_ORDER[v.order]},"
                f"{_GUARD[v.guard]},{r.ppc},{r.n},{r.t_prologue_ns},{r.t_compute_ns},"
                f"{r.t_epilogue_ns},{r.t_total_ns},{r.ns_per_update:.3f}\n")
    return out
