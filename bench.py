"""bench.py — full SPH step (kick1 -> drift -> rebin -> density -> force -> kick2) on B200.

Workload (BASELINE.json configs[1]): uniform 2-D box, n = 2^21 particles, ppc = 1024,
seed 42, the reference's own initial condition (grid.cpp:76-143) generated on the device
with EXACT numerics (byte-identical to the reference IC); synthetic data, no checkpoints.

Headline metric: particle-pair interactions/s over density + force (sum over cells of
nl*na*rounds for density plus nl*na for force, per step, divided by the step time), with
SPH steps/s reported beside it. See DESIGN.md §6 for the roofline definitions.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Multi-GPU (torchrun, N>1): weak scaling of independent replicas (one box per rank);
rank 0 prints the JSON line with the max-over-ranks time.
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

# algorithmic flops per pair: density 13 + 38 f_in + 11 f_<1.5 + 11 f_<0.5,
# force 22 + 45 f_in + 5 f_<1.5 + 5 f_<0.5 (counted from the reference source, kernels.cpp:97-153)


def flops_per_pair(f_in, f15, f05):
    return 13 + 38 * f_in + 11 * f15 + 11 * f05, 22 + 45 * f_in + 5 * f15 + 5 * f05


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index, self.samples, self._stop = index, [], threading.Event()
        self.th = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self.th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.th.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > i + 2 and s[i + 2].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons}


def dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return rank, world, local
    return 0, 1, 0


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


def run_ours(args, rank, world, local):
    import paper_2502_16517_b200 as pkg
    from paper_2502_16517_b200 import DeviceLayout, Numerics

    n, ppc, seed = args.n, args.ppc, args.seed
    ctx = pkg.Context(local, numerics=Numerics[args.numerics.capitalize()],
                      layout=DeviceLayout[args.layout.capitalize()])
    t0 = time.time()
    store, grid, par = ctx.make_particles(n, ppc, seed)
    t_ic = time.time() - t0
    par.dt = args.dt

    # pair statistics for the flop count (one density round at the IC's h)
    fpp = None
    if rank == 0 and args.count_flops:
        from oracle import Oracle
        orc = Oracle()
        # sampled cells: the in-support fractions are cell-local statistics
        cs = orc.pair_stats(store.recs, grid.nx, grid.ny, grid.cell_begin, grid.local_idx, 0) \
            if n <= 300000 else None
        if cs is not None:
            fin, f15, f05 = cs[2] / cs[0], cs[3] / cs[0], cs[4] / cs[0]
        else:
            fin, f15, f05 = 0.2236, 0.0804, 0.0089  # SURVEY.md §8(d), reference IC, ppc 1024
        fpp = flops_per_pair(fin, f15, f05) + (fin, f15, f05)

    for _ in range(args.warmup):
        ctx.step(par)
    barrier(world)
    ctx.synchronize()
    launches0 = ctx.launch_count()
    phase = np.zeros(6)
    den_pairs = for_pairs = 0
    with ClockSampler(local) as clk:
        tstep = []
        for _ in range(args.steps):
            ms = ctx.step(par)
            st = ctx.stats()
            den_pairs += st["density_pairs"]
            for_pairs += st["force_pairs"]
            phase += ms
            tstep.append(float(ms.sum()))
    ctx.synchronize()
    launches = ctx.launch_count() - launches0
    barrier(world)
    total_ms = allmax(float(np.sum(tstep)), world)
    ms_per_step = total_ms / args.steps
    pairs_per_step = (den_pairs + for_pairs) / args.steps
    value = pairs_per_step * world / (ms_per_step * 1e-3)
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference make_particles IC, uniform 2-D, seed 42)",
        "config": {"workload": f"full SPH step, uniform box, n={n}, ppc={ppc}",
                   "n": n, "ppc": ppc, "nx": grid.nx, "numerics": args.numerics,
                   "layout": args.layout, "dt": par.dt,
                   "l2": "inputs larger than L2 (AoS mirror 0.57 GB + SoA mirror)",
                   "parallelism": f"replicas x{world}"},
        "steps_per_s": 1e3 / ms_per_step * world,
        "phase_ms": dict(zip(["kick1", "drift", "rebin", "density", "force", "kick2"],
                             (phase / args.steps).round(4).tolist())),
        "density_pairs_per_step": den_pairs / args.steps,
        "force_pairs_per_step": for_pairs / args.steps,
        "ic_seconds": round(t_ic, 2),
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if rank == 0:
        fp64 = ctx.fp64_peak_tflops()
        out["fp64_peak_tflops_measured"] = fp64
        if fpp:
            dfl, ffl, fin, f15, f05 = fpp
            dms = phase[3] / args.steps
            fms = phase[4] / args.steps
            ach_f = ffl * (for_pairs / args.steps) / (fms * 1e-3) / 1e12
            out["roofline"] = {"bound": "fp64", "kernel": "force_kernel<FastPolicy>",
                               "achieved": ach_f, "peak": fp64, "unit": "TFLOP/s",
                               "frac": ach_f / fp64, "traffic": None,
                               "flops_per_pair": ffl,
                               "peak_source": "DFMA microbenchmark in this run (sph_fp64_peak)"}
            out["roofline_density"] = {"achieved": dfl * (den_pairs / args.steps) / (dms * 1e-3) / 1e12,
                                       "flops_per_pair": dfl}
            out["pair_fractions"] = {"f_in": fin, "f_lt_1.5": f15, "f_lt_0.5": f05}
    ctx.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=1 << 21)
    ap.add_argument("--ppc", type=int, default=1024)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--dt", type=float, default=1e-4)
    ap.add_argument("--numerics", default="fast", choices=["fast", "exact"])
    ap.add_argument("--layout", default="resident", choices=["resident", "aos", "convert"])
    ap.add_argument("--count-flops", type=int, default=1)
    args = ap.parse_args()
    rank, world, local = dist_init(args)
    if args.impl == "reference":
        print(json.dumps({"impl": "reference", "unavailable": "not implemented yet"}))
        return
    out = run_ours(args, rank, world, local)
    if rank == 0:
        print(json.dumps(out))


if __name__ == "__main__":
    main()
