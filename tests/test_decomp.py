"""Slab domain decomposition (paper_2502_16517_b200/decomp.py), world sizes 2-4 over gloo.

The host-side logic (partition, migration, halo exchange, owned-cell sweeps) is checked
on CPU with the oracle as the compute backend: k ranks must reproduce the single-rank
reference step byte for byte. The GPU variant runs the same logic with the device backend
(two processes sharing one GPU, gloo for the exchange).
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2502_16517_b200.decomp import (DistributedSim, Exchanger, SlabDecomposition,
                                          balanced_bounds, cell_of, column_costs)

N, PPC, SEED, DT, STEPS = 6000, 64, 4, 1e-2, 3


class OracleBackend:
    """Test-only compute backend: the CPU oracle restatement."""

    def __init__(self):
        from oracle import Oracle
        self.orc = Oracle()

    def linear(self, kernel, recs, ranks, par):
        n = len(recs)
        self.orc.sweep(kernel, recs, 1, 1, 1.0, np.array([0, n], np.int64), np.arange(n, dtype=np.int64), par)

    def pair(self, kernel, recs, ranks, nx, ny, mask, par):
        c = cell_of(recs, nx, ny)
        cb = np.zeros(nx * ny + 1, np.int64)
        np.cumsum(np.bincount(c, minlength=nx * ny), out=cb[1:])
        self.orc.sweep_masked(kernel, recs, nx, ny, 1.0 / nx, cb, np.arange(len(recs), dtype=np.int64),
                              par, mask)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def decomposition(recs, nx, world, rank, balanced):
    """Equal column counts, or (balanced) slabs of near-equal pair work from the IC."""
    if not balanced:
        return SlabDecomposition(nx, nx, world, rank)
    counts = np.bincount(cell_of(recs, nx, nx), minlength=nx * nx)
    return SlabDecomposition(nx, nx, world, rank, col_cost=column_costs(counts, nx, nx))


def reference_run(orc, recs, par):
    r = recs.copy()
    nx = orc.grid_nx(len(r), PPC)
    for _ in range(STEPS):
        for k in (3, 2):
            cb, li = orc.build_grid(r, nx)
            orc.sweep(k, r, nx, nx, 1.0 / nx, cb, li, par)
        cb, li = orc.build_grid(r, nx)
        for k in (0, 1, 4):
            orc.sweep(k, r, nx, nx, 1.0 / nx, cb, li, par)
    return r


def _worker(rank, world, port, out_path, use_gpu, kind=0, balanced=False):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    from oracle import Oracle
    from paper_2502_16517_b200 import Numerics, SphParams
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    orc = Oracle()
    orc.threads = 2
    recs, par = orc.make_particles(N, PPC, SEED, kind=kind)
    par = SphParams(dt=DT, gamma=par.gamma, cfl=par.cfl, grav=par.grav,
                    target_wcount=par.target_wcount)
    nx = orc.grid_nx(N, PPC)
    d = decomposition(recs, nx, world, rank, balanced)
    own, ranks = DistributedSim.split_global(recs, d)
    if use_gpu:
        from paper_2502_16517_b200.decomp import DeviceBackend
        be = DeviceBackend(0, numerics=Numerics.Exact)
    else:
        be = OracleBackend()
        be.orc.threads = 2
    sim = DistributedSim(d, own, ranks, be, Exchanger())
    for _ in range(STEPS):
        sim.step(par)
    out = sim.gather()
    if rank == 0:
        np.save(out_path, out)
    dist.barrier()
    dist.destroy_process_group()


def _run(world, use_gpu, kind=0, balanced=False):
    port = _free_port()
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "out.npy")
        mp.spawn(_worker, args=(world, port, out, use_gpu, kind, balanced), nprocs=world, join=True)
        return np.load(out)


def test_slab_geometry():
    d = SlabDecomposition(17, 17, 3, 1)
    assert list(d.owned_cols()) == list(range(5, 11))
    assert list(d.halo_cols()) == [4, 11]
    assert d.neighbours() == [0, 2]
    assert list(d.send_cols(0)) == [5] and list(d.send_cols(2)) == [10]
    d0 = SlabDecomposition(17, 17, 3, 0)
    assert list(d0.halo_cols()) == [5, 16]  # torus wrap
    m = d.owned_cells_mask()
    assert m.sum() == 6 * 17 and m[5] and not m[4]
    with pytest.raises(ValueError):
        SlabDecomposition(5, 5, 3, 0)


def test_split_partitions_every_particle(orc):
    recs, _ = orc.make_particles(3000, 64, 2)
    nx = orc.grid_nx(3000, 64)
    seen = []
    for r in range(3):
        own, ranks = DistributedSim.split_global(recs, SlabDecomposition(nx, nx, 3, r))
        seen.append(ranks)
    allr = np.sort(np.concatenate(seen))
    assert np.array_equal(allr, np.arange(3000))


@pytest.mark.parametrize("world,kind,balanced", [(2, 0, False), (3, 0, False), (4, 0, False),
                                                 (2, 1, False), (3, 1, True), (4, 0, True)])
def test_decomposed_steps_equal_single_rank(orc, world, kind, balanced):
    """world ranks (gloo, oracle compute; compact halo records: 40 B before density, 64 B
    before force) == the single-rank reference, byte for byte: uniform and clustered
    (variable ppc) boxes, equal-column and pair-work-balanced slabs."""
    from paper_2502_16517_b200 import SphParams
    recs, par = orc.make_particles(N, PPC, SEED, kind=kind)
    par = SphParams(dt=DT, gamma=par.gamma, cfl=par.cfl, grav=par.grav,
                    target_wcount=par.target_wcount)
    ref = reference_run(orc, recs, par)
    assert np.count_nonzero(ref["cell"] != recs["cell"]) > 0  # particles changed cells
    got = _run(world, use_gpu=False, kind=kind, balanced=balanced)
    assert got.tobytes() == ref.tobytes()


def test_balanced_bounds_even_out_pair_work(orc):
    """On a clustered box the pair-work-balanced slabs differ from equal columns and spread
    the pair work more evenly; on equal costs they are the equal-column slabs."""
    recs, _ = orc.make_particles(20000, 64, 3, kind=1)
    nx = orc.grid_nx(20000, 64)
    cost = column_costs(np.bincount(cell_of(recs, nx, nx), minlength=nx * nx), nx, nx)
    for world in (2, 4):
        eq = [(r * nx) // world for r in range(world + 1)]
        bb = balanced_bounds(cost, world)
        spread = lambda b: max(cost[b[r]:b[r + 1]].sum() for r in range(world)) / (cost.sum() / world)
        assert spread(bb) <= spread(eq)
        assert all(bb[r + 1] - bb[r] >= 2 for r in range(world))
    assert balanced_bounds(np.ones(128), 8) == [16 * r for r in range(9)]


@pytest.mark.gpu
def test_decomposed_steps_on_device_equal_single_rank(orc):
    """Same, with the device backend (EXACT) for both ranks on one GPU."""
    from paper_2502_16517_b200 import SphParams
    recs, par = orc.make_particles(N, PPC, SEED)
    par = SphParams(dt=DT, gamma=par.gamma, cfl=par.cfl, grav=par.grav,
                    target_wcount=par.target_wcount)
    ref = reference_run(orc, recs, par)
    got = _run(2, use_gpu=True)
    assert got.tobytes() == ref.tobytes()


def _dev_worker(rank, world, port, out_path, numerics_name, kind=0, balanced=False):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    from paper_2502_16517_b200 import Context, DeviceLayout, Numerics
    from paper_2502_16517_b200.decomp import DeviceSlabSim
    if world > 1:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
    torch.cuda.set_device(0)
    ctx = Context(0, numerics=Numerics[numerics_name], layout=DeviceLayout.Resident)
    par = ctx.make_particles_device(N, PPC, SEED, kind=kind)
    par.dt = DT
    import math
    nx = max(1, int(math.floor(1.0 / math.sqrt(PPC / N))))  # grid.cpp:23-26
    cost = column_costs(ctx.cell_counts(), nx, nx) if balanced else None
    d = SlabDecomposition(nx, nx, world, rank, col_cost=cost)
    DeviceSlabSim.start(ctx, d)
    sim = DeviceSlabSim(ctx, d)
    for _ in range(STEPS):
        sim.step(par)
    recs, ranks = sim.gather_sorted()
    if rank == 0:
        assert np.array_equal(ranks, np.arange(N))
        np.save(out_path, recs)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    ctx.close()


def _run_dev(world, numerics_name, kind=0, balanced=False):
    port = _free_port()
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "out.npy")
        mp.spawn(_dev_worker, args=(world, port, out, numerics_name, kind, balanced),
                 nprocs=world, join=True)
        return np.load(out)


@pytest.mark.gpu
def test_device_resident_decomposition_exact_equals_reference(orc):
    """Device-resident slabs (sph_dd_*: migration, halo records and rho refresh moved as
    device buffers), 2 ranks sharing one GPU over gloo, EXACT numerics: byte-identical to
    the CPU reference step."""
    from paper_2502_16517_b200 import SphParams
    recs, par = orc.make_particles(N, PPC, SEED)
    par = SphParams(dt=DT, gamma=par.gamma, cfl=par.cfl, grav=par.grav,
                    target_wcount=par.target_wcount)
    ref = reference_run(orc, recs, par)
    got = _run_dev(2, "Exact")
    assert got.tobytes() == ref.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("world,kind,balanced", [(2, 0, False), (3, 0, False), (4, 0, False),
                                                 (2, 1, False), (4, 1, True)])
def test_device_resident_decomposition_fast_equals_one_rank(world, kind, balanced):
    """FAST numerics: k device-resident ranks == one rank, byte for byte (each owned cell
    sees the same active list in the same order, so even the reassociated FAST sums agree;
    the interior / boundary force split runs the same per-cell work), uniform and clustered
    boxes, equal-column and pair-work-balanced slabs."""
    one = _run_dev(1, "Fast", kind)
    many = _run_dev(world, "Fast", kind, balanced)
    assert many.tobytes() == one.tobytes()


@pytest.mark.parametrize("nx,world", [(9, 2), (17, 3), (45, 4), (128, 8), (90, 4)])
def test_device_slab_masks_are_consistent(nx, world):
    """The column masks DeviceSlabSim moves buffers with: what rank r sends to q is exactly
    what q expects from r (halo and rho refresh), the migration targets cover every column
    outside the slab that a one-column move can reach, and the slabs partition the grid."""
    from paper_2502_16517_b200.decomp import DeviceSlabSim
    ms = [DeviceSlabSim.masks(SlabDecomposition(nx, nx, world, r)) for r in range(world)]
    assert np.array_equal(sum(m["mine"].astype(int) for m in ms), np.ones(nx, int))
    for r, m in enumerate(ms):
        for q in m["peers"]:
            assert r in ms[q]["peers"]
            assert np.array_equal(m["send_to"][q], ms[q]["halo_from"][r])
            assert not np.any(m["send_to"][q] & ~m["mine"].astype(bool))
            assert np.array_equal(m["cols_of"][q], ms[q]["mine"])
        # the columns adjacent to the slab (where a migrating particle can land) belong to peers
        cols = np.nonzero(m["mine"])[0]
        for c in ((cols[0] - 1) % nx, (cols[-1] + 1) % nx):
            assert any(m["cols_of"][q][c] for q in m["peers"])
    # the force split: interior + boundary = owned cells; no interior cell touches a halo column
    for r in range(world):
        d = SlabDecomposition(nx, nx, world, r)
        inner, bnd = DeviceSlabSim.force_split(d)
        own = d.owned_cells_mask().astype(np.uint8)
        assert np.array_equal(inner + bnd, own) and not np.any(inner & bnd)
        halo = set(d.halo_cols().tolist())
        for c in np.nonzero(inner)[0]:
            cx = c % nx
            assert not ({(cx - 1) % nx, cx, (cx + 1) % nx} & halo)
