"""Host-side mirror of the reference's L0 data types.

* ``PARTICLE_DTYPE`` — the packed 272-byte AoS ``Particle`` record
  (reference ``include/soaview/sph/particle.hpp:11-46``; offsets pinned by its
  ``static_assert``s and re-checked in ``tests/test_layout_contract.py``).
* ``SphParams`` — EOS / step constants (``particle.hpp:49-55``).
* ``KernelId`` / ``Path`` / ``Order`` / ``Guard`` / ``Layout`` — the reference's sweep
  selectors (``kernels.hpp:9-20``, ``grid.hpp:15``), same integer values.
* ``KernelTimes`` — per-phase times returned by ``run_sweep`` (``kernels.hpp:24-29``).
"""
from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

RECORD_SIZE = 272

PARTICLE_DTYPE = np.dtype(
    {
        "names": [
            "x", "v", "v_pred", "a", "m", "rho", "p", "u", "u_pred", "u_dt", "c", "h",
            "wcount", "rho_dh", "rot_v", "div_v", "v_sig", "h_dt", "dt_next", "frozen",
            "moved", "id", "cell", "flags", "dbg", "spare",
        ],
        "formats": [
            ("<f8", (2,)), ("<f8", (2,)), ("<f8", (2,)), ("<f8", (2,)), "<f8", "<f8", "<f8",
            "<f8", "<f8", "<f8", "<f8", "<f8", "<f8", "<f8", "<f8", "<f8", "<f8", "<f8", "<f8",
            "<i4", "<i4", "<i8", "<i8", "<i8", ("<f8", (2,)), ("<f8", (5,)),
        ],
        "offsets": [
            0, 16, 32, 48, 64, 72, 80, 88, 96, 104, 112, 120, 128, 136, 144, 152, 160, 168,
            176, 184, 188, 192, 200, 208, 216, 232,
        ],
        "itemsize": RECORD_SIZE,
    }
)
assert PARTICLE_DTYPE.itemsize == RECORD_SIZE


class KernelId(enum.IntEnum):
    Density = 0
    Force = 1
    Drift = 2
    Kick1 = 3
    Kick2 = 4


class Path(enum.IntEnum):
    AosBaseline = 0
    SoaView = 1


class Order(enum.IntEnum):
    LocalActive = 0
    ActiveLocal = 1


class Guard(enum.IntEnum):
    Branch = 0
    Mask = 1


class Layout(enum.IntEnum):
    """Host storage variant (grid.hpp:15)."""
    Scattered = 0
    Continuous = 1


class DeviceLayout(enum.IntEnum):
    """Device-side layout mode per sweep (the layout ablation, BASELINE.json config 4)."""
    FromPath = -1   # AosBaseline -> Aos, SoaView -> Convert (the C++ shim's mapping)
    Aos = 0         # kernels read/write the 272-B AoS mirror in place
    Convert = 1     # per-call AoS->SoA gather, SoA compute, SoA->AoS scatter
    Resident = 2    # SoA mirror stays resident; AoS materialised on download


class Numerics(enum.IntEnum):
    Exact = 0       # reference op order, no FMA, IEEE sqrt/div: byte-identical results
    Fast = 1        # FMA + rsqrt/Newton + hoisting; parity within stated tolerance


@dataclass
class SphParams:
    dt: float = 1.0e-4
    gamma: float = 5.0 / 3.0
    cfl: float = 0.1
    grav: float = 1.0
    target_wcount: float = 0.0

    def as_array(self) -> np.ndarray:
        return np.array([self.dt, self.gamma, self.cfl, self.grav, self.target_wcount],
                        dtype=np.float64)

    @classmethod
    def from_array(cls, a) -> "SphParams":
        return cls(*[float(v) for v in a[:5]])


@dataclass
class KernelTimes:
    prologue_ns: int = 0
    compute_ns: int = 0
    epilogue_ns: int = 0

    def total(self) -> int:
        return self.prologue_ns + self.compute_ns + self.epilogue_ns


def empty_particles(n: int) -> np.ndarray:
    return np.zeros(n, dtype=PARTICLE_DTYPE)
