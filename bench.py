"""bench.py — full SPH step (kick1 -> drift -> rebin -> density -> force -> kick2) on B200.

Workload (BASELINE.json configs[1]): uniform 2-D periodic box, n = 2^21 particles,
ppc = 1024 (nx = 45, 2025 cells), seed 42 — the reference's own initial condition
(make_particles, grid.cpp:76-143), generated on the device with EXACT numerics
(byte-identical to the reference IC, tests/test_gpu_parity.py). Synthetic data.

Metric: particle-pair interactions/s over density + force. The pair count of the workload
is implementation-independent: sum over cells of nl*na for density plus the same for
force (one pass each, kernels.cpp:204-303), per step, divided by the step time; extra
h-iteration rounds (kernels.cpp:184-192) are work the step has to do, not extra credit.
SPH steps/s is reported beside it.

  value  : device-resident step (state stays in HBM), CUDA events on the library stream
  e2e    : the same step through the C-ABI on HOST records (sph_step_host): every step
           copies all records host->device and device->host (pinned host memory)
  roofline: force kernel (largest share of the step) vs the FP64 pipe peak measured
           live by a DFMA microbenchmark (sph_fp64_peak); HBM kernels beside it
  cpu_baseline: the unmodified reference (oracle/_ref) on this host's cores, one full step
           from the same state (oracle/ref_bench.py)
  --impl reference: the same reference, full steps, nothing of this repo's CUDA loaded

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
N>1 (torchrun): weak scaling, --particles per GPU of one global box slab-decomposed
over the GPUs (device-resident slabs, NCCL migration / halo / rho exchange each step,
decomp.DeviceSlabSim); time = device events around the K steps, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particle-pair interactions/sec (density+force)"
UNIT = "pairs/s"
IC_KIND = {"uniform": 0, "clustered": 1}  # clustered = BASELINE config 3 (sph_b200.h)


def flops_per_pair(f_in, f15, f05):
    """Algorithmic flops per evaluated pair counted from the reference source
    (SURVEY.md §8(d)): density 13 + 38 f_in + 11 f_<1.5 + 11 f_<0.5,
    force 22 + 45 f_in + 5 f_<1.5 + 5 f_<0.5."""
    return 13 + 38 * f_in + 11 * f15 + 11 * f05, 22 + 45 * f_in + 5 * f15 + 5 * f05


# bytes per particle the resident-SoA streaming kernels move: their view descriptors'
# fields in + out (kernels.cpp:808-859), drift 52+28, kick1 48+32, kick2 104+80 (the SoA
# mirror holds dbg[0] only, so kick2 reads 8 B less than its 112-B descriptor)
LINEAR_BYTES = {"kick1": 80, "drift": 80, "kick2": 184}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def captured_workload(args):
    """The committed ncu capture (tools/profile.sh) is of the default workload: BASELINE
    config 2, 2^21 particles, ppc 1024, uniform IC, FAST numerics, resident layout."""
    return (args.n, args.ppc, args.ic, args.numerics, args.layout) == (
        1 << 21, 1024, "uniform", "fast", "resident")


def load_pipe(kernel, args):
    """FP64-pipe activity (%) of a kernel from the committed ncu capture (its workload only)."""
    if not captured_workload(args):
        return None
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return {"pct": d["kernels"][kernel]["fp64_pipe_active_pct"], "source": d.get("source", p)}
    except Exception:
        return None


def load_traffic(args):
    """dram bytes per launch of the force kernel from the committed ncu capture; null for any
    workload other than the captured one."""
    if not captured_workload(args):
        return None, "not captured for this workload (the ncu capture is of config 2)"
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        k = d["kernels"].get("force2_kernel") or d["kernels"]["force_kernel<FastPolicy>"]
        return k["dram_bytes_read"] + k["dram_bytes_write"], d.get("source", p)
    except Exception:
        return None, None


class ClockSampler:
    """SM clocks + throttle reasons sampled (NVML, every 20 ms) during the timed region;
    falls back to nvidia-smi polling if pynvml is unavailable."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index=0):
        self.index, self.samples, self._stop = index, [], threading.Event()
        self.th = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((float(sm), float(mx),
                                     sorted(k for k, b in self.REASONS.items() if r & b)))
                self._stop.wait(0.02)
            return
        except Exception:
            pass
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        names = ["hw_slowdown", "sw_thermal_slowdown", "hw_thermal_slowdown", "sw_power_cap"]
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip().split(",")
                v = [x.strip() for x in out]
                self.samples.append((float(v[0]), float(v[1]),
                                     [names[i] for i in range(4) if v[i + 2].lower() == "active"]))
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self.th.start()
        t0 = time.time()  # the timed region starts only once sampling is running
        while not self.samples and self.th.is_alive() and time.time() - t0 < 5.0:
            time.sleep(0.005)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.th.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted({r for s in self.samples for r in s[2]}),
                "samples": len(self.samples)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        if os.environ.get("SPH_BENCH_SHARE_GPU") == "1":
            # functional check of the N>1 path on a one-GPU box: every rank on GPU 0, gloo
            # (host-staged) exchanges; the timings of such a run mean nothing
            local = 0
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allmax(v, world):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def config_block(args, nx, world):
    box = ("uniform 2-D box" if args.ic == "uniform" else
           "clustered 2-D box (variable ppc: half uniform, half in 16 Gaussian clumps)")
    return {"workload": f"full SPH step, {box}, n={args.n}, ppc={args.ppc}", "ic": args.ic,
            "n": args.n, "ppc": args.ppc, "nx": nx, "seed": args.seed,
            "dt": args.dt, "numerics": args.numerics, "layout": args.layout,
            "l2": (f"inputs larger than L2 (AoS mirror {272 * args.n / 1e9:.2f} GB + SoA mirror "
                   f"~{210 * args.n / 1e9:.2f} GB)"),
            "parallelism": "single GPU"}


def grid_nx(n, ppc):
    """grid.cpp:23-26."""
    import math
    return max(1, int(math.floor(1.0 / math.sqrt(ppc / max(n, 1)))))


def run_decomposed(args, rank, world, local):
    """N > 1 GPUs: weak scaling. One global box of N * args.n particles (the reference IC,
    nx = floor(sqrt(N n / ppc))) is cut into N slabs of cell columns; each GPU keeps its
    slab on the device and exchanges migration records, halo records and the halo rho
    refresh with its two neighbours over NCCL every step (decomp.DeviceSlabSim). Time:
    device events around K steps, max over ranks."""
    import torch
    import torch.distributed as dist

    import paper_2502_16517_b200 as pkg
    from paper_2502_16517_b200 import DeviceLayout, Numerics
    from paper_2502_16517_b200.decomp import DeviceSlabSim, SlabDecomposition, column_costs

    ctx = pkg.Context(local, numerics=Numerics[args.numerics.capitalize()],
                      layout=DeviceLayout.Resident)
    n_glob = args.n if args.strong else args.n * world
    t0 = time.time()
    par = ctx.make_particles_device(n_glob, args.ppc, args.seed, kind=IC_KIND[args.ic])
    par.dt = args.dt
    nx = grid_nx(n_glob, args.ppc)
    # slabs of near-equal pair work (sum of nl * na per column) of the global IC, which
    # every rank holds identically at this point
    d = SlabDecomposition(nx, nx, world, rank, col_cost=column_costs(ctx.cell_counts(), nx, nx))
    DeviceSlabSim.start(ctx, d)
    sim = DeviceSlabSim(ctx, d)
    t_ic = time.time() - t0
    dev = torch.device("cuda", local)
    dist.barrier()  # first collective on every rank before the point-to-point batches

    def total(v, op=dist.ReduceOp.SUM):
        t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=op)
        return float(t.item())

    for _ in range(args.warmup):
        sim.step(par)
    workload_pairs = total(2 * ctx.stats()["active_pairs"])
    n_local = ctx.count()
    torch.cuda.synchronize()
    dist.barrier()
    launches0 = ctx.launch_count()
    sent0 = sim.bytes_sent
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    den = forc = 0.0
    with ClockSampler(local) as clk:
        e0.record()
        for _ in range(args.steps):
            sim.step(par)
            den += ctx.stats()["last_density_ms"]
            forc += sim.force_ms
        e1.record()
        torch.cuda.synchronize()
    dist.barrier()
    ms_total = total(e0.elapsed_time(e1), dist.ReduceOp.MAX)
    ms_per_step = ms_total / args.steps
    launches = ctx.launch_count() - launches0
    out = {
        "metric": METRIC, "value": workload_pairs / (ms_per_step * 1e-3), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong" if args.strong else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: reference make_particles IC of the global box (uniform random 2-D, "
                "seed 42), generated on each device, byte-identical to the reference",
        "config": {"workload": f"full SPH step, {n_glob // world} particles per GPU, global box of "
                               f"{n_glob} particles (nx={nx}), ppc={args.ppc}, slab decomposition",
                   "ic": args.ic, "n": n_glob, "n_per_gpu": n_glob // world, "ppc": args.ppc, "nx": nx,
                   "seed": args.seed, "dt": args.dt, "numerics": args.numerics,
                   "layout": "resident",
                   "l2": "inputs larger than L2 (>= 1 GB of mirrors per GPU)",
                   "slab_bounds": d.bounds,
                   "parallelism": f"slab decomposition x{world} (NCCL halo + migration, "
                                  f"pair-work-balanced slabs)"},
        "steps_per_s": 1e3 / ms_per_step,
        "workload_pairs_per_step": workload_pairs,
        "phase_ms": {"density": den / args.steps, "force": forc / args.steps},
        "exchange_bytes_per_step_rank0": (sim.bytes_sent - sent0) / args.steps,
        "ic_seconds": round(t_ic, 2),
        "gpu_launches": launches,
        "gpu_launches_per_step": launches / args.steps,
        "clocks": clk.summary(),
    }
    # e2e: the rank's owned records come from pinned host memory before every step and go
    # back after it (sph_dd_append / sph_dd_export through the C-ABI)
    e2e_steps = args.steps if args.e2e_steps is None else args.e2e_steps
    if e2e_steps > 0:
        allm = np.ones(nx, np.uint8)
        host = torch.empty(n_local * 272 + 4096, dtype=torch.uint8, pin_memory=True)
        hrank = torch.empty(n_local + 16, dtype=torch.int64, pin_memory=True)
        wall = []
        for it in range(e2e_steps + 1):
            dist.barrier()
            t1 = time.perf_counter()
            if it > 0:  # host -> device: replace the device state with the host records
                m = hrank_n
                recs_d = host[: m * 272].to(dev, non_blocking=True)
                ranks_d = hrank[:m].to(dev, non_blocking=True)
                torch.cuda.synchronize()
                ctx.dd_remove(allm)
                ctx.dd_append(recs_d.data_ptr(), ranks_d.data_ptr(), m)
            sim.step(par)
            recs_d, ranks_d = sim._export(allm)  # device -> host: the step's result
            hrank_n = ranks_d.numel()
            if hrank_n * 272 > host.numel():
                host = torch.empty(hrank_n * 272 + 4096, dtype=torch.uint8, pin_memory=True)
                hrank = torch.empty(hrank_n + 16, dtype=torch.int64, pin_memory=True)
            host[: hrank_n * 272].copy_(recs_d)
            hrank[:hrank_n].copy_(ranks_d)
            torch.cuda.synchronize()
            if it > 0:
                wall.append(time.perf_counter() - t1)
        e2e_s = total(float(np.mean(wall)), dist.ReduceOp.MAX)
        nb = total(n_local * 272, dist.ReduceOp.MAX)
        out["e2e"] = {"value": workload_pairs / e2e_s, "unit": UNIT,
                      "h2d_bytes_per_step": int(nb), "d2h_bytes_per_step": int(nb),
                      "ms_per_step": e2e_s * 1e3, "steps": e2e_steps,
                      "api": "per rank: H2D of the owned records (sph_dd_append), the "
                             "decomposed step, D2H of the owned records (sph_dd_export)"}
    ctx.close()
    return out if rank == 0 else None


def run_ours(args, rank, world, local):
    # N > 1 is the slab-decomposed box; a failure there is reported as a failure (no
    # fallback to independent replicas, which would not be the workload)
    if world > 1:
        return run_decomposed(args, rank, world, local)
    return run_single(args, rank, world, local)


def run_single(args, rank, world, local):
    import paper_2502_16517_b200 as pkg
    from paper_2502_16517_b200 import DeviceLayout, Numerics

    ctx = pkg.Context(local, numerics=Numerics[args.numerics.capitalize()],
                      layout=DeviceLayout[args.layout.capitalize()])
    t0 = time.time()
    store, grid, par = ctx.make_particles(args.n, args.ppc, args.seed, kind=IC_KIND[args.ic])
    t_ic = time.time() - t0
    par.dt = args.dt
    workload_pairs = 2 * ctx.stats()["active_pairs"]

    # ---- device-resident timed region ----
    for _ in range(args.warmup):
        ctx.step(par)
    ctx.synchronize()
    barrier(world)
    launches0 = ctx.launch_count()
    phase = np.zeros(6)
    den_eval = 0
    round_ms = np.zeros(4)
    steps_ms = []
    mid_state = None  # the CPU baseline times the middle step of the timed range
    with ClockSampler(local) as clk:
        for it in range(args.steps):
            if it == args.steps // 2 and world == 1 and args.cpu_baseline:
                mid_state = ctx.read_records()  # between steps: outside the device-event time
            ms = ctx.step(par)
            st = ctx.stats()
            den_eval += st["density_pairs"]
            round_ms += np.array(st["density_round_ms"])
            phase += ms
            steps_ms.append(float(ms.sum()))
    args.mid_state = mid_state
    args.mid_step = args.warmup + args.steps // 2 + 1
    ctx.synchronize()
    launches = ctx.launch_count() - launches0
    barrier(world)
    total_ms = allmax(float(np.sum(steps_ms)), world)
    ms_per_step = total_ms / args.steps
    value = workload_pairs * world / (ms_per_step * 1e-3)
    ph = phase / args.steps
    names = ["kick1", "drift", "rebin", "density", "force", "kick2"]

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: reference make_particles IC (uniform random 2-D, seed 42), "
                "generated on device, byte-identical to the reference",
        "config": config_block(args, grid.nx, world),
        "steps_per_s": 1e3 / ms_per_step * world,
        "workload_pairs_per_step": workload_pairs,
        "density_pairs_evaluated_per_step": den_eval / args.steps,
        "phase_ms": dict(zip(names, ph.round(4).tolist())),
        "density_round_kernel_ms": (round_ms / args.steps).round(4).tolist(),
        "ic_seconds": round(t_ic, 2),
        "gpu_launches": launches,
        "gpu_launches_per_step": launches / args.steps,
        "clocks": clk.summary(),
    }

    # ---- e2e: the same step through the C-ABI on pinned host records ----
    e2e_steps = args.steps if args.e2e_steps is None else args.e2e_steps
    if e2e_steps <= 0:
        return _finish(out, ctx, store, grid, par, args, rank, world, ph, names, den_eval,
                       workload_pairs)
    # the host records still hold the initial condition: the end-to-end run repeats the
    # device run's trajectory, W warm-up steps then the timed ones (steps W+1 .. W+E), so
    # `value`, `e2e` and the reference arm all time the same simulated steps (the density work
    # grows with simulated time)
    ctx.host_register(store.recs)
    try:
        for _ in range(args.warmup):
            ctx.step_host(par)
        barrier(world)
        wall = []
        dev = np.zeros(8)
        for _ in range(e2e_steps):
            t0 = time.perf_counter()
            dev += ctx.step_host(par)
            wall.append(time.perf_counter() - t0)
        barrier(world)
    finally:
        ctx.host_unregister(store.recs)
    e2e_s = allmax(float(np.mean(wall)), world)
    nbytes = store.recs.nbytes
    out["e2e"] = {"value": workload_pairs * world / e2e_s, "unit": UNIT,
                  "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
                  "ms_per_step": e2e_s * 1e3, "steps": e2e_steps,
                  "api": "sph_step_host (C-ABI, host Particle records in and out)",
                  "trajectory": (f"from the initial condition, {args.warmup} warm-up steps, "
                                 f"timed steps {args.warmup + 1}-{args.warmup + e2e_steps} "
                                 f"(the device run times steps {args.warmup + 1}-"
                                 f"{args.warmup + args.steps})"),
                  "device_ms": dict(zip(["h2d"] + names + ["d2h"],
                                        (dev / e2e_steps).round(3).tolist()))}
    return _finish(out, ctx, store, grid, par, args, rank, world, ph, names, den_eval,
                   workload_pairs)


def _finish(out, ctx, store, grid, par, args, rank, world, ph, names, den_eval, workload_pairs):
    if rank == 0:
        fp64 = ctx.fp64_peak_tflops()
        peaks, src = load_peaks()
        # exact support fractions of the final state: a device counting pass with the
        # reference's arithmetic, outside the timed region (sph_pair_fractions)
        fin, f15, f05, _ = ctx.pair_fractions()
        dfl, ffl = flops_per_pair(fin, f15, f05)
        fpairs = workload_pairs / 2
        ach_f = ffl * fpairs / (ph[4] * 1e-3) / 1e12
        ach_d = dfl * (den_eval / args.steps) / (ph[3] * 1e-3) / 1e12
        traffic, tsrc = load_traffic(args)
        out["roofline"] = {
            "bound": "fp64", "kernel": "force2_kernel", "achieved": ach_f,
            "peak": fp64, "unit": "TFLOP/s", "frac": ach_f / fp64, "traffic": traffic,
            "traffic_source": tsrc,
            "flops_per_pair": ffl, "pairs_per_launch": fpairs, "launch_ms": ph[4],
            "peak_source": "FP64 DFMA microbenchmark run in this process (sph_fp64_peak); "
                           "nominal 37.2 TFLOP/s at 1965 MHz",
            "note": "force evaluates gravity on every active pair (nothing culled), so this "
                    "is bounded by the FP64 pipe",
        }
        pipe_f = load_pipe("force2_kernel", args)
        if pipe_f is not None:  # the hardware view beside the algorithmic-flop one
            out["roofline"]["fp64_pipe_pct_ncu"] = pipe_f
        cull_note = ("effective: the reference's algorithmic flops for every active pair "
                     "(SURVEY 8(d)); density skips chunks out of the warp's reach, so on "
                     "clustered boxes this can exceed the pipe peak; not pipe utilisation")
        out["roofline_density"] = {"achieved": ach_d, "frac": ach_d / fp64,
                                   "flops_per_pair": dfl, "unit": "TFLOP/s", "note": cull_note}
        # pipe-honest companions: (1) only the flops of pairs the kernel certainly evaluates
        # in full (the in-support ones; the distance tests of evaluated out-of-support pairs
        # are not counted, so this is a lower bound), (2) ncu's measured FP64-pipe activity
        ins = (dfl - 13.0 * (1.0 - fin)) * (den_eval / args.steps)
        ach_i = ins / (ph[3] * 1e-3) / 1e12
        out["roofline_density"]["in_support_only"] = {
            "achieved": ach_i, "frac": ach_i / fp64, "flops_per_step": ins,
            "note": "flops of the in-support pairs only (every one is evaluated); a lower bound "
                    "of the work done, beside the 'effective' figure above, an upper one"}
        pipe = load_pipe("density2_kernel", args)
        if pipe is not None:
            out["roofline_density"]["fp64_pipe_pct_ncu"] = pipe
        # the north-star figure: the whole step (density rounds + force + linear kernels +
        # rebin) against the FP64 pipe, algorithmic flops of the pair sweeps per step
        step_flops = dfl * (den_eval / args.steps) + ffl * fpairs
        ach_s = step_flops / (float(np.sum(ph)) * 1e-3) / 1e12
        out["roofline_step"] = {"achieved": ach_s, "peak": fp64, "frac": ach_s / fp64,
                                "unit": "TFLOP/s", "flops_per_step": step_flops,
                                "ms_per_step": float(np.sum(ph)), "note": cull_note}
        hbm = peaks.get("hbm_gbs", 6650.0)
        out["roofline_linear"] = {
            k: {"achieved_gbs": LINEAR_BYTES[k] * args.n / (ph[names.index(k)] * 1e-3) / 1e9,
                "bytes_per_particle": LINEAR_BYTES[k],
                "peak_gbs": hbm, "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({src})",
                "frac": LINEAR_BYTES[k] * args.n / (ph[names.index(k)] * 1e-3) / 1e9 / hbm,
                "note": "effective: bytes the kernel's fields occupy / kernel time; the peak "
                        "is a copy (half reads, half writes), which a read-heavy kernel can "
                        "exceed slightly"}
            for k in LINEAR_BYTES}
        out["pair_fractions"] = {"f_in": fin, "f_lt_1.5": f15, "f_lt_0.5": f05,
                                 "source": "exact device count of the final state "
                                           "(sph_pair_fractions, reference arithmetic)"}
        if world == 1 and args.cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(ctx, store, grid, par, args)
    ctx.close()
    return out


def _host_state(ctx, store):
    """Current device state as host records (for statistics and the CPU baseline)."""
    import paper_2502_16517_b200 as pkg
    recs = ctx.read_records()
    return pkg.ParticleStore(recs, np.arange(len(recs), dtype=np.int64), pkg.Layout.Continuous)


def cpu_baseline(ctx, store, grid, par, args):
    """One full reference step (oracle/_ref) of the middle step of the timed range (the state
    the device run had there; the density work grows with simulated time), on all host cores,
    wall clock; rank 0 at N = 1 only."""
    from oracle.ref_bench import ReferenceStepper
    recs = getattr(args, "mid_state", None)
    if recs is None:
        recs = _host_state(ctx, store).recs
    stepper = ReferenceStepper(recs, args.ppc, par.as_array(), sample_pairs=args.cpu_sample_pairs)
    t = stepper.step()
    frac = t["sample_fraction"]
    what = ("density and force on every cell" if frac >= 1.0 else
            f"density and force on {100 * frac:.1f}% of the pair work, random cells, scaled by "
            f"pair count")
    return {"value": t["workload_pairs"] / t["step"], "unit": UNIT,
            "cores": stepper.threads, "kind": "reference",
            "step_seconds": t["step"], "measured_seconds": t["measured_seconds"],
            "sample": f"one full reference step (kick1, drift, build_grid, kick2 on all {args.n} "
                      f"particles; {what}) of the same workload: simulated step "
                      f"{getattr(args, 'mid_step', '?')}, the middle of the timed range; "
                      f"oracle/_ref built from /root/reference; wall clock",
            "phase_seconds": {k: round(t[k], 4) for k in
                              ("kick1", "drift", "rebin", "density", "force", "kick2")}}


def _loaded_native_libs():
    """Shared objects of this repo mapped into the process (for the reference arm's
    self-check: it must not load libsph_b200.so)."""
    try:
        with open("/proc/self/maps") as f:
            paths = {ln.split()[-1] for ln in f if ln.rstrip().endswith(".so")}
    except OSError:
        return []
    return sorted(os.path.relpath(p, ROOT) for p in paths if p.startswith(ROOT))


def run_reference(args, rank, world, local):
    """The reference's own CPU implementation (oracle/_ref, the unmodified reference sources
    compiled by oracle/Makefile) on this host's cores: full steps (kick1, drift, build_grid,
    density, force, kick2 through the reference's run_sweep / build_grid on every cell),
    wall clock. Nothing of this repo's CUDA library is loaded on this arm."""
    if rank != 0:
        return None
    from oracle import Oracle, ref_available
    from oracle.ref_bench import ReferenceStepper
    if not ref_available():
        return {"impl": "reference", "unavailable": "oracle/_ref was not built (needs /root/reference)"}
    # IC: the reference make_particles (grid.cpp:76-143) as restated by oracle/liboracle.so,
    # threaded and byte-identical to the reference's own (tests/test_oracle.py); the
    # reference's single-threaded make_particles needs ~4 min at 2^21. Outside the timed region.
    t0 = time.time()
    recs, par = Oracle().make_particles(args.n, args.ppc, args.seed, kind=IC_KIND[args.ic])
    t_ic = time.time() - t0
    par.dt = args.dt
    stepper = ReferenceStepper(recs, args.ppc, par.as_array(), sample_pairs=args.ref_sample_pairs)
    for _ in range(args.warmup):
        stepper.step()
    ts = [stepper.step() for _ in range(args.steps)]
    step_s = float(np.mean([t["step"] for t in ts]))
    pairs = ts[0]["workload_pairs"]
    v = pairs / step_s
    frac = ts[0]["sample_fraction"]
    sample = ("each step: the full reference step (kick1, drift, build_grid, density, force, "
              "kick2) on every cell and particle" if frac >= 1.0 else
              f"each step: linear kernels + build_grid on all particles, density/force on "
              f"{100 * frac:.1f}% of the pair work (random cells), scaled by pair count")
    libs = _loaded_native_libs()
    assert not any("libsph_b200" in p for p in libs), libs
    return {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: reference make_particles IC (uniform random 2-D, seed 42)",
        "config": config_block(args, grid_nx(args.n, args.ppc), 1),
        "steps_per_s": 1.0 / step_s,
        "workload_pairs_per_step": pairs,
        "phase_seconds": {k: round(float(np.mean([t[k] for t in ts])), 4)
                          for k in ("kick1", "drift", "rebin", "density", "force", "kick2")},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": stepper.threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "ic_seconds": round(t_ic, 2),
        "native_libs_loaded": libs,
        "gpu_launches": 0,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--particles", dest="n", type=int, default=1 << 21,
                    help="particles (per GPU when --gpus > 1)")
    ap.add_argument("--ppc", type=int, default=1024)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--dt", type=float, default=1e-4)
    ap.add_argument("--numerics", default="fast", choices=["fast", "exact"])
    ap.add_argument("--ic", default="uniform", choices=["uniform", "clustered"])
    ap.add_argument("--layout", default="resident", choices=["resident", "aos", "convert"])
    ap.add_argument("--e2e-steps", type=int, default=None,
                    help="timed end-to-end steps (default: --steps, after --warmup warm-up "
                         "steps from the initial condition: the device run's trajectory)")
    ap.add_argument("--strong", action="store_true",
                    help="N > 1: --particles is the global box (BASELINE config 5 strong scaling) "
                         "instead of the per-GPU count (weak scaling, the default)")
    ap.add_argument("--cpu-baseline", type=int, default=1)
    ap.add_argument("--cpu-sample-pairs", type=float, default=None,
                    help="cpu_baseline: restrict density/force to ~x pairs of random cells "
                         "(default: the full reference step)")
    ap.add_argument("--ref-sample-pairs", type=float, default=None,
                    help="--impl reference: as --cpu-sample-pairs (default: full steps)")
    args = ap.parse_args()
    rank, world, local = dist_init()
    if args.impl == "reference":
        out = run_reference(args, rank, world, local)
    else:
        out = run_ours(args, rank, world, local)
    if rank == 0 and out is not None:
        print(json.dumps(out))


if __name__ == "__main__":
    main()
