"""Spatial domain decomposition of the SPH step across ranks.

The reference has no decomposition; this is the B200 build's multi-GPU path,
designed so that EXACT results on k ranks equal 1 rank equal the CPU reference:

* ``SlabDecomposition``: the periodic nx x ny cell grid is cut into slabs of cell columns,
  one per rank. A rank owns the particles of its columns and keeps a one-column halo on
  each side (torus wrap). Halo particles keep their GLOBAL cell and ParticleStore::all
  rank, so every owned cell sees exactly the reference's active list (build_grid order,
  grid.cpp:152-182).
* ``DistributedSim.step``: kick1 + drift on owned particles -> migration of particles that
  left the slab (272-B records to their new owner) -> halo exchange of boundary-column
  records -> density on owned cells -> halo refresh (density changed rho, which force
  reads for active particles, kernels.cpp:443-456) -> force on owned cells -> kick2.
  Exchanges are point-to-point with the two slab neighbours (``torch.distributed``: NCCL
  on GPUs, gloo in the CPU tests).
* Compute goes through a backend: ``DeviceBackend`` (the C-ABI, one context per rank) in
  production; tests plug in the CPU oracle to check the host-side logic on any machine.
"""
from __future__ import annotations

import numpy as np

from .particle import PARTICLE_DTYPE, RECORD_SIZE, DeviceLayout, KernelId, Numerics, SphParams

DENSITY, FORCE, DRIFT, KICK1, KICK2 = (int(k) for k in (KernelId.Density, KernelId.Force,
                                                         KernelId.Drift, KernelId.Kick1,
                                                         KernelId.Kick2))


def cell_of(recs: np.ndarray, nx: int, ny: int) -> np.ndarray:
    """build_grid's cell index (grid.cpp:153-155): clamp(floor(x*nx)), row-major."""
    x = recs["x"]
    cx = np.clip(np.floor(x[:, 0] * nx).astype(np.int64), 0, nx - 1)
    cy = np.clip(np.floor(x[:, 1] * nx).astype(np.int64), 0, ny - 1)
    return cy * nx + cx


def column_costs(counts: np.ndarray, nx: int, ny: int) -> np.ndarray:
    """Pair work of each cell column: sum over its cells of nl * na, na = the locals of the
    wrapped, deduplicated 3x3 stencil (grid.cpp:159-182), from per-cell local counts."""
    nl = np.asarray(counts, np.float64).reshape(ny, nx)
    seen, na = set(), np.zeros_like(nl)
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            key = (dy % ny, dx % nx)
            if key not in seen:
                seen.add(key)
                na += np.roll(np.roll(nl, -dy, axis=0), -dx, axis=1)
    return (nl * na).sum(axis=0)


def balanced_bounds(col_cost: np.ndarray, world: int) -> list[int]:
    """Column bounds of `world` slabs with near-equal pair work: slab r ends at the first
    column where the cumulative cost reaches (r + 1) / world of the total; every slab keeps
    at least two columns."""
    nx = len(col_cost)
    cum = np.cumsum(np.asarray(col_cost, np.float64))
    tot = cum[-1] if nx else 0.0
    b = [0]
    for r in range(1, world):
        if tot > 0:  # end the slab at the column boundary closest to the target share
            t = r * tot / world
            k = int(np.searchsorted(cum, t, side="left"))  # cum[k] >= t
            below = cum[k - 1] if k > 0 else 0.0
            c = k + 1 if cum[min(k, nx - 1)] - t <= t - below else k
        else:
            c = (r * nx) // world
        c = max(c, b[-1] + 2)
        c = min(c, nx - 2 * (world - r))
        b.append(c)
    b.append(nx)
    return b


class SlabDecomposition:
    """Slabs of cell columns of the periodic nx x ny grid; rank r owns [c0_r, c1_r).

    Without ``col_cost`` the slabs have equal column counts; with it (``column_costs`` of
    the particle distribution) they have near-equal pair work (variable-ppc boxes)."""

    def __init__(self, nx: int, ny: int, world: int, rank: int, col_cost=None):
        if world < 1 or not 0 <= rank < world:
            raise ValueError("bad world / rank")
        if world > 1 and nx < 2 * world:
            raise ValueError("each rank needs at least two cell columns")
        self.nx, self.ny, self.world, self.rank = nx, ny, world, rank
        if col_cost is None:
            self.bounds = [(r * nx) // world for r in range(world + 1)]
        else:
            if len(col_cost) != nx:
                raise ValueError("col_cost needs one entry per column")
            self.bounds = balanced_bounds(col_cost, world)
        self.col_owner = np.empty(nx, np.int64)
        for r in range(world):
            self.col_owner[self.bounds[r]:self.bounds[r + 1]] = r

    def owned_cols(self, r: int | None = None) -> np.ndarray:
        r = self.rank if r is None else r
        return np.arange(self.bounds[r], self.bounds[r + 1])

    def halo_cols(self, r: int | None = None) -> np.ndarray:
        r = self.rank if r is None else r
        if self.world == 1:
            return np.zeros(0, np.int64)
        c0, c1 = self.bounds[r], self.bounds[r + 1]
        h = {(c0 - 1) % self.nx, c1 % self.nx}
        return np.array(sorted(c for c in h if self.col_owner[c] != r), np.int64)

    def neighbours(self) -> list[int]:
        return sorted({int(self.col_owner[c]) for c in self.halo_cols()} - {self.rank})

    def cells_mask(self, cols: np.ndarray) -> np.ndarray:
        m = np.zeros(self.nx, bool)
        m[cols] = True
        return np.tile(m, self.ny)

    def owned_cells_mask(self) -> np.ndarray:
        return self.cells_mask(self.owned_cols())

    def send_cols(self, q: int) -> np.ndarray:
        """My owned columns that lie in rank q's halo."""
        return np.intersect1d(self.owned_cols(), self.halo_cols(q))


class Exchanger:
    """Neighbour point-to-point exchange of (records, all_rank) sets; records of any
    structured dtype (whole 272-B records for migration, compact halo records)."""

    def __init__(self, group=None, device=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.device = device  # None: CPU tensors (gloo); else a torch.device (NCCL)
        self.bytes_sent = 0

    def exchange(self, send: dict[int, tuple[np.ndarray, np.ndarray]], peers: list[int],
                 dtype=PARTICLE_DTYPE):
        import torch
        dist = self.dist
        dev = self.device or torch.device("cpu")
        cnt_in = {q: torch.zeros(1, dtype=torch.int64, device=dev) for q in peers}
        reqs = []
        for q in peers:
            n = len(send.get(q, (np.zeros(0, dtype),))[0])
            reqs.append(dist.isend(torch.tensor([n], dtype=torch.int64, device=dev), q, group=self.group))
            reqs.append(dist.irecv(cnt_in[q], q, group=self.group))
        for r in reqs:
            r.wait()
        reqs, bufs = [], {}
        keep = []
        for q in peers:
            recs, ranks = send.get(q, (np.zeros(0, dtype), np.zeros(0, np.int64)))
            if len(recs):
                t = torch.from_numpy(np.ascontiguousarray(recs, dtype).view(np.uint8).reshape(-1)).to(dev)
                tr = torch.from_numpy(np.ascontiguousarray(ranks, np.int64)).to(dev)
                keep += [t, tr]
                self.bytes_sent += t.numel() + 8 * tr.numel()
                reqs.append(dist.isend(t, q, group=self.group))
                reqs.append(dist.isend(tr, q, group=self.group))
            m = int(cnt_in[q].item())
            if m:
                b = torch.empty(m * np.dtype(dtype).itemsize, dtype=torch.uint8, device=dev)
                br = torch.empty(m, dtype=torch.int64, device=dev)
                bufs[q] = (b, br)
                reqs.append(dist.irecv(b, q, group=self.group))
                reqs.append(dist.irecv(br, q, group=self.group))
        for r in reqs:
            r.wait()
        out = {}
        for q in peers:
            if q in bufs:
                b, br = bufs[q]
                out[q] = (b.cpu().numpy().view(dtype).copy(), br.cpu().numpy().copy())
            else:
                out[q] = (np.zeros(0, dtype), np.zeros(0, np.int64))
        return out


class DeviceBackend:
    """Sweeps through the C-ABI on this rank's GPU (host-staged: records are bound per call)."""

    def __init__(self, device: int = 0, numerics: Numerics = Numerics.Fast):
        from .sph import Context
        self.ctx = Context(device, numerics=numerics, layout=DeviceLayout.Resident)

    def _bind(self, recs, ranks, nx, ny, mask=None):
        from .sph import CellGrid, ParticleStore
        store = ParticleStore(recs, np.arange(len(recs), dtype=np.int64))
        if mask is None:  # linear kernels: any grid enumerating every particle once
            grid = CellGrid(1, 1, 1.0, np.array([0, len(recs)], np.int64),
                            np.arange(len(recs), dtype=np.int64), store,
                            all_rank=np.asarray(ranks, np.int64))
        else:
            c = cell_of(recs, nx, ny)
            cb = np.zeros(nx * ny + 1, np.int64)
            np.cumsum(np.bincount(c, minlength=nx * ny), out=cb[1:])
            grid = CellGrid(nx, ny, 1.0 / nx, cb, np.arange(len(recs), dtype=np.int64), store,
                            all_rank=np.asarray(ranks, np.int64))
        self.ctx.bind(grid)
        if mask is not None:
            self.ctx.set_owned_cells(mask)

    def linear(self, kernel: int, recs, ranks, par):
        if len(recs):
            self._bind(recs, ranks, 1, 1)
            self.ctx.run_sweep(KernelId(kernel), par)

    def pair(self, kernel: int, recs, ranks, nx, ny, owned_mask, par):
        """recs must be sorted by (cell, all_rank)."""
        if len(recs):
            self._bind(recs, ranks, nx, ny, owned_mask)
            self.ctx.run_sweep(KernelId(kernel), par)

    def close(self):
        self.ctx.close()


def sort_local(recs, ranks, nx, ny):
    """(cell, all_rank) order = build_grid's list order for the global store."""
    c = cell_of(recs, nx, ny)
    order = np.lexsort((ranks, c))
    return recs[order], ranks[order]


class DistributedSim:
    """One rank of the slab-decomposed leapfrog step."""

    def __init__(self, decomp: SlabDecomposition, recs: np.ndarray, ranks: np.ndarray,
                 backend, exchanger: Exchanger | None):
        self.d = decomp
        self.own = np.ascontiguousarray(recs)
        self.ranks = np.ascontiguousarray(ranks, np.int64)
        self.be = backend
        self.ex = exchanger
        self.last = {}

    @staticmethod
    def split_global(recs: np.ndarray, decomp: SlabDecomposition):
        """This rank's owned share of a global store (records in ParticleStore::all order)."""
        c = cell_of(recs, decomp.nx, decomp.ny)
        mine = decomp.col_owner[c % decomp.nx] == decomp.rank
        return recs[mine].copy(), np.nonzero(mine)[0].astype(np.int64)

    # Fields a pair sweep reads from an active particle that is not one of its locals
    # (kernels.cpp:379-392, :443-456): density x, v_pred, m (40 B); force also rho, p, c (64 B).
    HALO_FIELDS = {DENSITY: ("x", "v_pred", "m"), FORCE: ("x", "v_pred", "m", "rho", "p", "c")}

    def _halo(self, kernel):
        d = self.d
        if d.world == 1:
            return np.zeros(0, PARTICLE_DTYPE), np.zeros(0, np.int64)
        cols = cell_of(self.own, d.nx, d.ny) % d.nx
        # only the kernel's active-view fields travel (a compact record); received halo
        # records are expanded with every other field zero
        fields = self.HALO_FIELDS[kernel]
        hdt = np.dtype([(f, PARTICLE_DTYPE.fields[f][0]) for f in fields])
        send = {}
        for q in d.neighbours():
            sel = np.isin(cols, d.send_cols(q))
            recs = np.zeros(int(sel.sum()), hdt)
            for f in fields:
                recs[f] = self.own[f][sel]
            send[q] = (recs, self.ranks[sel])
        got = self.ex.exchange(send, d.neighbours(), dtype=hdt)
        recs, rk = [], []
        for q in d.neighbours():
            h = np.zeros(len(got[q][0]), PARTICLE_DTYPE)
            for f in fields:
                h[f] = got[q][0][f]
            recs.append(h)
            rk.append(got[q][1])
        return np.concatenate(recs) if recs else np.zeros(0, PARTICLE_DTYPE), \
            np.concatenate(rk) if rk else np.zeros(0, np.int64)

    def _migrate(self):
        d = self.d
        if d.world == 1:
            return
        dest = d.col_owner[cell_of(self.own, d.nx, d.ny) % d.nx]
        stay = dest == d.rank
        peers = d.neighbours()
        if np.any(~stay & ~np.isin(dest, peers)):
            raise RuntimeError("a particle moved more than one slab in one step")
        send = {q: (self.own[dest == q], self.ranks[dest == q]) for q in peers}
        got = self.ex.exchange(send, peers)
        self.own = np.concatenate([self.own[stay]] + [got[q][0] for q in peers])
        self.ranks = np.concatenate([self.ranks[stay]] + [got[q][1] for q in peers])

    def _pair(self, kernel, par):
        d = self.d
        hrecs, hranks = self._halo(kernel)
        n_own = len(self.own)
        recs = np.concatenate([self.own, hrecs])
        ranks = np.concatenate([self.ranks, hranks])
        is_own = np.zeros(len(recs), bool)
        is_own[:n_own] = True
        c = cell_of(recs, d.nx, d.ny)
        order = np.lexsort((ranks, c))
        recs, ranks, is_own = recs[order], ranks[order], is_own[order]
        self.be.pair(kernel, recs, ranks, d.nx, d.ny, d.owned_cells_mask(), par)
        self.own, self.ranks = recs[is_own].copy(), ranks[is_own].copy()

    def step(self, par: SphParams):
        self.be.linear(KICK1, self.own, self.ranks, par)
        self.be.linear(DRIFT, self.own, self.ranks, par)
        self._migrate()
        # build_grid writes p->cell for every particle (grid.cpp:156)
        self.own["cell"] = cell_of(self.own, self.d.nx, self.d.ny)
        self._pair(DENSITY, par)  # halo carries x, v_pred, m (and p, c from the last kick2)
        self._pair(FORCE, par)    # fresh halo: rho updated by the owners' density
        self.be.linear(KICK2, self.own, self.ranks, par)

    def gather(self, group=None):
        """All owned particles on every rank, in global ParticleStore::all order (tests)."""
        import torch
        import torch.distributed as dist
        if self.d.world == 1:
            order = np.argsort(self.ranks)
            return self.own[order]
        objs = [None] * self.d.world
        dist.all_gather_object(objs, (self.own, self.ranks), group=group)
        recs = np.concatenate([o[0] for o in objs])
        ranks = np.concatenate([o[1] for o in objs])
        return recs[np.argsort(ranks)]


class DeviceSlabSim:
    """One rank of the DEVICE-RESIDENT slab decomposition (BASELINE config 5).

    The rank's context holds its slab's particles on its GPU for the whole run. Per step:

    1. kick1 + drift;
    2. migration: whole records (272 B + all-rank) of the particles whose column left the
       slab go to the neighbour that owns it (``sph_dd_export`` assembles them from the SoA
       mirror; ``sph_dd_append`` puts them straight into it);
    3. halo: each neighbour gets my particles in its halo columns as 56-B halo records,
       x, v_pred, m (density's active fields, kernels.cpp:379-392) plus p and c (force's,
       which kick2 last set) and the all-rank (``sph_dd_export_halo`` /
       ``sph_dd_append_halo``); rebin; density on the owned cells;
    4. rho of the halo (8 B per halo particle; force reads the active particles' rho,
       kernels.cpp:443-456): the send is posted, force runs on the interior cells (whose
       3x3 stencil holds no halo column) while it is in flight, then rho is imported and
       force runs on the boundary cells. The counts are the halo counts of step 3, so this
       exchange needs no count round and, over NCCL, no host synchronisation;
    5. kick2, drop the halo.

    Transport: ``torch.distributed`` point-to-point with the two slab neighbours: NCCL over
    NVLink between GPUs (the context then runs on torch's current stream, so the NCCL
    kernels are ordered with its sweeps), gloo in the CPU-staged tests. Owned cells see
    exactly the reference's active lists (halo particles keep their global cell and
    all-rank), so k ranks reproduce one rank byte for byte.
    """

    def __init__(self, ctx, decomp: SlabDecomposition, group=None):
        import torch
        self.ctx, self.d, self.group = ctx, decomp, group
        self.torch = torch
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.nccl = False
        if decomp.world > 1:
            import torch.distributed as dist
            self.dist = dist
            self.nccl = dist.get_backend(group) == "nccl"
        if self.nccl:  # one stream for the sweeps and the NCCL ordering
            ctx.set_stream(torch.cuda.current_stream(self.dev).cuda_stream)
        m = self.masks(decomp)
        self.mine, self.not_mine, self.peers = m["mine"], m["not_mine"], m["peers"]
        self.cols_of, self.send_to, self.halo_from = m["cols_of"], m["send_to"], m["halo_from"]
        self.interior, self.boundary = self.force_split(decomp)
        self.bytes_sent = 0
        self.force_ms = 0.0
        self.halo_out, self.halo_in = {}, {}

    @staticmethod
    def masks(decomp: SlabDecomposition) -> dict:
        """Column masks (nx bytes) of one rank: its own columns, the rest, and per neighbour
        q the columns q owns (migration), my columns in q's halo (halo / rho send) and my
        halo columns owned by q (halo / rho receive)."""
        nx = decomp.nx
        mine = np.zeros(nx, np.uint8)
        mine[decomp.owned_cols()] = 1
        out = {"mine": mine, "not_mine": (1 - mine).astype(np.uint8),
               "peers": decomp.neighbours(), "cols_of": {}, "send_to": {}, "halo_from": {}}
        for q in out["peers"]:
            for key, cols in (("cols_of", decomp.owned_cols(q)),
                              ("send_to", decomp.send_cols(q)),
                              ("halo_from", np.intersect1d(decomp.halo_cols(), decomp.owned_cols(q)))):
                mk = np.zeros(nx, np.uint8)
                mk[cols] = 1
                out[key][q] = mk
        return out

    @staticmethod
    def force_split(decomp: SlabDecomposition):
        """Owned cells (ncells bytes) whose 3x3 stencil holds no halo column (interior) and
        the rest of the owned cells (boundary)."""
        nx, ny = decomp.nx, decomp.ny
        own = np.zeros(nx, bool)
        own[decomp.owned_cols()] = True
        inner = own & np.roll(own, 1) & np.roll(own, -1)
        if decomp.world == 1:
            inner = own.copy()
        interior = np.tile(inner, ny).astype(np.uint8)
        boundary = np.tile(own & ~inner, ny).astype(np.uint8)
        return interior, boundary

    @staticmethod
    def start(ctx, decomp: SlabDecomposition) -> None:
        """Keep this rank's columns of a globally bound context and set the owned cells."""
        mine = np.zeros(decomp.nx, np.uint8)
        mine[decomp.owned_cols()] = 1
        if decomp.world > 1:
            ctx.dd_remove(1 - mine)
            ctx.rebin()
        ctx.set_owned_cells(decomp.owned_cells_mask().astype(np.uint8))

    # ---- transport ----
    def _exchange(self, sends: dict, counts_in: dict | None = None):
        """sends[q] = tuple of 1-D device tensors; returns the peers' tuples (same dtypes).
        counts_in[q] (element counts per tensor) skips the count round when known."""
        torch, dist = self.torch, self.dist
        stage = (lambda t: t) if self.nccl else (lambda t: t.cpu())
        home = self.dev if self.nccl else torch.device("cpu")
        first = next(iter(sends.values()))
        if counts_in is None:
            cnt_out = {q: torch.tensor([t.numel() for t in sends[q]], dtype=torch.int64, device=home)
                       for q in self.peers}
            cnt_in = {q: torch.zeros(len(first), dtype=torch.int64, device=home) for q in self.peers}
            ops = []
            for q in self.peers:
                ops.append(dist.P2POp(dist.isend, cnt_out[q], q, group=self.group))
                ops.append(dist.P2POp(dist.irecv, cnt_in[q], q, group=self.group))
            for r in dist.batch_isend_irecv(ops):
                r.wait()
            counts_in = {q: cnt_in[q].tolist() for q in self.peers}
        ops, recv, keep = [], {}, []
        for q in self.peers:
            bufs = []
            for t, m in zip(sends[q], counts_in[q]):
                if t.numel():
                    st = stage(t)
                    keep.append(st)
                    ops.append(dist.P2POp(dist.isend, st, q, group=self.group))
                    self.bytes_sent += st.numel() * st.element_size()
                b = torch.empty(int(m), dtype=t.dtype, device=home)
                if m:
                    ops.append(dist.P2POp(dist.irecv, b, q, group=self.group))
                bufs.append(b)
            recv[q] = bufs
        reqs = dist.batch_isend_irecv(ops) if ops else []
        return reqs, recv, keep

    def _finish(self, reqs, recv):
        for r in reqs:
            r.wait()  # NCCL: the current stream waits for the transfer (no host block)
        out = {q: tuple(b.to(self.dev) for b in recv[q]) for q in self.peers}
        self._sync_torch()
        return out

    def _sync_torch(self):
        """gloo: the context runs on its own stream, so torch's copies into / allocations of
        the buffers it reads must be complete first (over NCCL both share one stream)."""
        if not self.nccl:
            self.torch.cuda.synchronize()

    def _export(self, mask):
        torch = self.torch
        self._sync_torch()
        m = self.ctx.dd_count(mask)
        recs = torch.empty(max(m, 1) * RECORD_SIZE, dtype=torch.uint8, device=self.dev)
        ranks = torch.empty(max(m, 1), dtype=torch.int64, device=self.dev)
        got = self.ctx.dd_export(mask, recs.data_ptr(), ranks.data_ptr(), m)
        assert got == m
        return recs[: m * RECORD_SIZE], ranks[:m]

    def _export_halo(self, mask):
        torch = self.torch
        self._sync_torch()
        m = self.ctx.dd_count(mask)
        vals = torch.empty(max(m, 1) * 7, dtype=torch.float64, device=self.dev)
        ranks = torch.empty(max(m, 1), dtype=torch.int64, device=self.dev)
        got = self.ctx.dd_export_halo(mask, vals.data_ptr(), ranks.data_ptr(), m)
        assert got == m
        return vals[: 7 * m], ranks[:m]

    def _timed_force(self, par, mask):
        self.ctx.sweep_cells(KernelId.Force, par, mask)
        self.force_ms += self.ctx.stats()["last_force_ms"]

    # ---- the step ----
    def step(self, par: SphParams) -> None:
        ctx, d = self.ctx, self.d
        ctx.sweep(KernelId.Kick1, par)
        ctx.sweep(KernelId.Drift, par)
        if d.world > 1:
            # migration: particles whose column left the slab go to its owner
            leaving = ctx.dd_count(self.not_mine)
            sends = {q: self._export(self.cols_of[q]) for q in self.peers}
            if sum(int(s[1].numel()) for s in sends.values()) != leaving:
                raise RuntimeError("a particle moved more than one slab in one step")
            got = self._finish(*self._exchange(sends)[:2])
            ctx.dd_remove(self.not_mine)
            for q in self.peers:
                recs, ranks = got[q]
                if ranks.numel():
                    ctx.dd_append(recs.data_ptr(), ranks.data_ptr(), ranks.numel())
            # halo: my particles in each neighbour's halo columns, 56-B halo records
            sends = {q: self._export_halo(self.send_to[q]) for q in self.peers}
            self.halo_out = {q: int(sends[q][1].numel()) for q in self.peers}
            got = self._finish(*self._exchange(sends)[:2])
            self.halo_in = {q: int(got[q][1].numel()) for q in self.peers}
            for q in self.peers:
                vals, ranks = got[q]
                if ranks.numel():
                    ctx.dd_append_halo(vals.data_ptr(), ranks.data_ptr(), ranks.numel())
        ctx.rebin()
        ctx.sweep(KernelId.Density, par)
        self.force_ms = 0.0
        if d.world > 1:
            torch = self.torch
            sends = {}
            self._sync_torch()
            for q in self.peers:
                m = self.halo_out[q]
                buf = torch.empty(max(m, 1), dtype=torch.float64, device=self.dev)
                assert ctx.dd_export_rho(self.send_to[q], buf.data_ptr(), m) == m
                sends[q] = (buf[:m],)
            reqs, recv, keep = self._exchange(sends, {q: [self.halo_in[q]] for q in self.peers})
            if self.interior.any():  # overlaps the rho transfer (NCCL)
                self._timed_force(par, self.interior)
            got = self._finish(reqs, recv)
            for q in self.peers:
                ctx.dd_import_rho(self.halo_from[q], got[q][0].data_ptr(), got[q][0].numel())
            self._timed_force(par, self.boundary)
            del keep
        else:
            ctx.sweep(KernelId.Force, par)
            self.force_ms = ctx.stats()["last_force_ms"]
        ctx.sweep(KernelId.Kick2, par)
        if d.world > 1:
            ctx.dd_remove(self.not_mine)  # drop the halo

    def gather_sorted(self):
        """All owned records of every rank in all-rank order (tests)."""
        torch = self.torch
        recs, ranks = self._export(np.ones(self.d.nx, np.uint8))
        r = recs.cpu().numpy().view(PARTICLE_DTYPE)
        k = ranks.cpu().numpy()
        if self.d.world > 1:
            objs = [None] * self.d.world
            self.dist.all_gather_object(objs, (r, k), group=self.group)
            r = np.concatenate([o[0] for o in objs])
            k = np.concatenate([o[1] for o in objs])
        return r[np.argsort(k, kind="stable")], np.sort(k)
