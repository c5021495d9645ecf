"""Pins the CPU oracle (oracle/sph_oracle.c) before it is trusted as the GPU checker.

1. against the committed golden vectors made from the UNMODIFIED reference
   (tests/golden/make_golden.py), byte for byte;
2. against the reference itself (oracle/_ref) when that build is present;
3. against the reference's own known-answer tests (test_sph.cpp:92-125, 213-306).
"""
import glob
import os

import numpy as np
import pytest

from paper_2502_16517_b200 import PARTICLE_DTYPE, SphParams

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
KERNELS = ["density", "force", "drift", "kick1", "kick2"]


def _grid(orc, recs, ppc):
    nx = orc.grid_nx(len(recs), ppc)
    cb, li = orc.build_grid(recs, nx)
    return nx, cb, li


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "ic_*.npz"))))
def test_oracle_matches_golden(orc, path):
    d = np.load(path)
    n, ppc, seed = (int(v) for v in os.path.basename(path)[3:-4].split("_"))
    ic, par = orc.make_particles(n, ppc, seed)
    assert ic.tobytes() == d["ic"].tobytes(), "IC (make_particles) differs"
    assert par.as_array().tobytes() == d["par"].tobytes()
    for k, name in enumerate(KERNELS):
        r = d["ic"].copy()
        nx, cb, li = _grid(orc, r, ppc)
        orc.sweep(k, r, nx, nx, 1.0 / nx, cb, li, d["par"])
        assert r.tobytes() == d[name].tobytes(), f"{name} differs from the reference"


def test_oracle_multistep_matches_golden(orc):
    path = glob.glob(os.path.join(GOLDEN, "steps_*.npz"))[0]
    d = np.load(path)
    n, ppc, seed = (int(v) for v in os.path.basename(path)[6:-4].split("_"))
    r, p = d["ic"].copy(), d["par"]
    for _ in range(3):
        for k in (3, 2):
            nx, cb, li = _grid(orc, r, ppc)
            orc.sweep(k, r, nx, nx, 1.0 / nx, cb, li, p)
        nx, cb, li = _grid(orc, r, ppc)
        for k in (0, 1, 4):
            orc.sweep(k, r, nx, nx, 1.0 / nx, cb, li, p)
    assert np.count_nonzero(r["cell"] != d["ic"]["cell"]) > 0
    assert r.tobytes() == d["out"].tobytes()


def test_spline_matches_golden(orc):
    d = np.load(os.path.join(GOLDEN, "spline.npz"))
    w = np.array([orc.kernel_w(q) for q in d["q"]])
    dw = np.array([orc.kernel_dw(q) for q in d["q"]])
    assert w.tobytes() == d["w"].tobytes()
    assert dw.tobytes() == d["dw"].tobytes()


@pytest.mark.parametrize("n,ppc,seed", [(700, 64, 11), (2000, 128, 1), (90, 64, 2)])
def test_oracle_matches_reference_build(orc, ref, n, ppc, seed):
    """Restatement vs the reference compiled from /root/reference (oracle/_ref)."""
    a, pa = ref.make_particles(n, ppc, seed, layout=1)
    b, pb = orc.make_particles(n, ppc, seed)
    assert a.tobytes() == b.tobytes() and pa == pb
    for k in range(5):
        A, B = a.copy(), a.copy()
        g = ref.grid(A, ppc)
        g.run_sweep(k, pa, path=k % 2, order=(k // 2) % 2, guard=k % 2)  # variants are bitwise-equal
        nx, cb, li = _grid(orc, B, ppc)
        orc.sweep(k, B, nx, nx, 1.0 / nx, cb, li, pa)
        assert A.tobytes() == B.tobytes(), KERNELS[k]


def test_scattered_layout_same_values(ref):
    """test_sph.cpp:138-149: layouts differ in storage only."""
    a, _ = ref.make_particles(900, 64, 5, layout=0)
    b, _ = ref.make_particles(900, 64, 5, layout=1)
    a = np.sort(a, order="id")
    b = np.sort(b, order="id")
    assert a.tobytes() == b.tobytes()


# --- reference known answers (test_sph.cpp) on the oracle ---

def test_spline_integrates_to_one(orc):
    """test_sph.cpp:92-97 (Simpson quadrature of 2*pi*q*W(q))."""
    def simpson(a, b, n):
        h = (b - a) / n
        acc = orc.kernel_w(a) * a + orc.kernel_w(b) * b
        for i in range(1, n):
            q = a + i * h
            acc += q * orc.kernel_w(q) * (4.0 if i % 2 else 2.0)
        return acc * h / 3.0
    integral = 2.0 * np.pi * (simpson(0.0, 0.5, 2048) + simpson(0.5, 1.5, 4096) +
                              simpson(1.5, 2.5, 4096))
    assert integral == pytest.approx(1.0, rel=1e-8)


def test_spline_derivative_and_support(orc):
    """test_sph.cpp:99-125."""
    for q in np.arange(0.013, 2.6, 0.031):
        if min(abs(q - b) for b in (0.5, 1.5, 2.5)) < 1e-3:
            continue
        eps = 1e-6
        num = (orc.kernel_w(q + eps) - orc.kernel_w(q - eps)) / (2 * eps)
        assert orc.kernel_dw(q) == pytest.approx(num, rel=1e-5, abs=1e-9)
    assert orc.kernel_w(2.5) == 0.0 and orc.kernel_dw(2.5) == 0.0 and orc.kernel_dw(0.0) == 0.0
    ws = [orc.kernel_w(i * 3.0 / 10000) for i in range(10001)]
    assert all(b <= a for a, b in zip(ws, ws[1:])) and min(ws) >= 0.0


def _bp(x0, x1):
    p = np.zeros(1, PARTICLE_DTYPE)
    p["x"] = (x0, x1)
    p["m"], p["h"], p["rho"], p["p"], p["c"], p["u"], p["u_pred"] = 1.0, 0.3, 1.0, 1.0, 1.0, 1.0, 1.0
    p["dt_next"] = 1e30
    return p


def test_linear_known_answers(orc):
    """test_sph.cpp:213-265 on the oracle's drift_one / kick1_one / kick2_one."""
    par = SphParams(dt=0.5).as_array()
    p = _bp(1.0, 2.0)
    p["v_pred"], p["u"], p["u_dt"] = (2.0, -1.0), 4.0, 8.0
    orc.one("drift", p, par)
    assert tuple(p["x"][0]) == (2.0, 1.5) and p["u_pred"][0] == 6.0 and p["moved"][0] == 1
    p = _bp(0.5, 0.5)
    p["u"], p["u_dt"] = 2.0, 4.0
    orc.one("kick1", p, SphParams())
    assert p["u"][0] == 2.0 + 0.5 * 1e-4 * 4.0
    assert p["dt_next"][0] == min(0.005 / 1e-12, np.sqrt(0.005 / 1e-12))
    p = _bp(0.5, 0.5)
    p["u_dt"], p["rho"], p["v_sig"] = -30000.0, 2.0, 3.0
    orc.one("kick2", p, SphParams())
    g = 5.0 / 3.0
    assert p["u"][0] == 0.5 and p["c"][0] == np.sqrt(g * (g - 1.0) * 0.5)
    assert p["p"][0] == (g - 1.0) * 2.0 * 0.5 and p["h_dt"][0] == 0.0


def test_isolated_and_pair_known_answers(orc):
    """test_sph.cpp:267-306 on the oracle."""
    r = _bp(0.5, 0.5)
    r["m"] = 2.0
    nx, cb, li = _grid(orc, r, 64)
    par = SphParams(target_wcount=orc.kernel_w(0.0))
    orc.sweep(0, r, nx, nx, 1.0 / nx, cb, li, par)
    assert r["rho"][0] == 2.0 * orc.kernel_w(0.0) * (1 / 0.3) * (1 / 0.3)
    assert r["h"][0] == 0.3 and r["flags"][0] == 0
    r = np.concatenate([_bp(0.4, 0.5), _bp(0.6, 0.5)])
    r["id"] = (0, 1)
    nx, cb, li = _grid(orc, r, 64)
    par = SphParams(target_wcount=orc.kernel_w(0.0) + orc.kernel_w(0.2 / 0.3))
    orc.sweep(0, r, nx, nx, 1.0 / nx, cb, li, par)
    assert r["rho"][0] == r["rho"][1] > 0
    orc.sweep(1, r, nx, nx, 1.0 / nx, cb, li, par)
    assert r["a"][0, 0] == -r["a"][1, 0] != 0.0 and r["v_sig"][0] == r["v_sig"][1]


def test_clustered_ic_is_variable_and_deterministic(orc):
    """Builder-defined variable-ppc IC (BASELINE config 3): deterministic per seed, the
    first half identical in distribution to the reference IC, strong ppc contrast."""
    a, pa = orc.make_particles(20000, 64, 3, kind=1)
    b, pb = orc.make_particles(20000, 64, 3, kind=1)
    assert a.tobytes() == b.tobytes() and pa == pb
    nx = orc.grid_nx(20000, 64)
    cb, _ = orc.build_grid(a.copy(), nx)
    c = np.diff(cb)
    assert c.max() > 2.5 * c.mean() and c.sum() == 20000
    assert np.all(a["x"] >= 0.0) and np.all(a["x"] <= 1.0)
