"""Host-side contract checks (no GPU needed):

* the 272-byte record layout and the per-kernel access sets match the reference's view
  descriptors (kernels.cpp:741-859, Table 1 byte counts);
* libsph_b200.so loads and exports every symbol include/sph_b200.h declares, and the
  header's selector values equal the reference enums;
* the host mirror's build_grid equals the reference build_grid (local and active lists);
* the product path fails loudly without a GPU (no CPU fallback).
"""
import ctypes as C
import re

import numpy as np
import pytest

import paper_2502_16517_b200 as pkg
from paper_2502_16517_b200 import _lib
from paper_2502_16517_b200.particle import PARTICLE_DTYPE

# A_in / A_out byte counts of the reference descriptors (kernels.cpp:741-859)
VIEW_BYTES = {  # which: (in_bytes, out_bytes)
    0: (88, 48), 1: (40, 0), 2: (128, 40), 3: (64, 0), 4: (52, 28), 5: (48, 32), 6: (112, 80)}


def test_record_layout_matches_reference(ref):
    assert PARTICLE_DTYPE.itemsize == 272
    offs = {name: PARTICLE_DTYPE.fields[name][1] for name in PARTICLE_DTYPE.names}
    seen = set()
    for which in range(7):
        for off, size, d in ref.view_fields(which):
            names = [k for k, v in offs.items() if v == off]
            assert names, f"no field at offset {off}"
            assert PARTICLE_DTYPE.fields[names[0]][0].itemsize == size
            seen.add(names[0])
    assert {"x", "v_pred", "m", "h", "rho", "p", "c", "a", "frozen", "moved", "dbg"} <= seen


def test_view_byte_counts(ref):
    for which, (bin_, bout) in VIEW_BYTES.items():
        f = ref.view_fields(which)
        assert sum(s for _, s, d in f if d in (0, 2)) == bin_
        assert sum(s for _, s, d in f if d in (1, 2)) == bout


def test_library_exports_header_symbols():
    lib = _lib.load()
    declared = _lib.declared_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.sph_abi_version() == 1


def test_header_enums_match_reference():
    src = open(_lib.HEADER).read()
    vals = dict(re.findall(r"(SPH_[A-Z0-9_]+) = (-?\d+)", src))
    assert [int(vals[k]) for k in ("SPH_DENSITY", "SPH_FORCE", "SPH_DRIFT", "SPH_KICK1", "SPH_KICK2")] == [0, 1, 2, 3, 4]
    assert int(vals["SPH_PATH_SOA_VIEW"]) == pkg.Path.SoaView
    assert int(vals["SPH_ORDER_ACTIVE_LOCAL"]) == pkg.Order.ActiveLocal
    assert int(vals["SPH_GUARD_MASK"]) == pkg.Guard.Mask
    assert C.sizeof(_lib.SphParamsC) == 40 and C.sizeof(_lib.SphTimesC) == 24


def test_no_cpu_fallback_without_gpu():
    import os
    if os.path.exists("/dev/nvidia0"):
        pytest.skip("GPU present")
    with pytest.raises(pkg.SphError):
        pkg.Context(0)


@pytest.mark.parametrize("n,ppc,seed", [(2048, 64, 3), (60, 64, 9), (250, 64, 9), (5000, 128, 4)])
def test_host_build_grid_matches_reference(ref, orc, n, ppc, seed):
    recs, _ = orc.make_particles(n, ppc, seed)
    # perturb so some particles leave [0,1) (no re-wrap after drift, cells clamp)
    recs["x"][::97] += 0.004
    recs["x"][::89] -= 0.004
    a = recs.copy()
    g = ref.grid(a, ppc)
    cb_ref, li_ref = g.local_csr()
    acb_ref, ai_ref = g.active_csr()
    store = pkg.ParticleStore(recs, np.arange(n, dtype=np.int64), pkg.Layout.Continuous)
    grid = pkg.build_grid(store, pkg.InitConfig(n=n, ppc=ppc))
    assert grid.nx == g.nx and grid.ny == g.ny and grid.cell_size == g.cell_size
    assert np.array_equal(grid.cell_begin, cb_ref) and np.array_equal(grid.local_idx, li_ref)
    assert np.array_equal(recs["cell"], a["cell"])
    for c in range(grid.cells()):
        assert np.array_equal(grid.active(c), ai_ref[acb_ref[c]:acb_ref[c + 1]])


def test_build_grid_respects_all_order(ref):
    """Local lists follow ParticleStore::all order (grid.cpp:152-158), not storage order."""
    rng = np.random.default_rng(0)
    n = 3000
    recs = np.zeros(n, PARTICLE_DTYPE)
    recs["x"] = rng.random((n, 2))
    order = rng.permutation(n)
    store = pkg.ParticleStore(recs, order.astype(np.int64), pkg.Layout.Scattered)
    grid = pkg.build_grid(store, pkg.InitConfig(n=n, ppc=64))
    g = ref.grid(recs.copy(), 64, order=order)
    cb, li = g.local_csr()
    assert np.array_equal(grid.local_idx, li)
    # all_rank is the rank in `all` of each local entry
    assert np.array_equal(order[grid.all_rank], grid.local_idx)
