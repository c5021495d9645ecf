"""The CPU-baseline driver (oracle/ref_bench.py) runs the reference step on a sample."""
import numpy as np
import pytest


def test_reference_stepper_small(orc, ref):
    from oracle.ref_bench import ReferenceStepper, stencil_pairs
    recs, par = orc.make_particles(3000, 64, 2)
    g = ref.grid(recs.copy(), 64)
    cb, _ = g.local_csr()
    per = stencil_pairs(cb, g.nx, g.ny)
    acb, ai = g.active_csr()
    assert np.array_equal(per, np.diff(cb) * np.diff(acb))
    st = ReferenceStepper(recs, 64, par.as_array(), threads=2, sample_pairs=1e6)
    t = st.step()
    assert t["workload_pairs"] == 2 * int(per.sum())
    assert 0 < t["sample_fraction"] <= 1.0
    for k in ("kick1", "drift", "rebin", "density", "force", "kick2", "step"):
        assert t[k] >= 0.0
