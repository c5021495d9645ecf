"""paper_2502_16517_b200 — B200-native (sm_100a) SPH particle kernels of arXiv 2502.16517.

Drop-in for the reference's SPH hot path (``soaview::sph::run_sweep`` and friends):
density / force neighbour sweeps over cell lists and the drift / kick1 / kick2 updates,
computed by hand-written CUDA kernels behind the C-ABI in ``include/sph_b200.h``.
"""
from .particle import (PARTICLE_DTYPE, RECORD_SIZE, DeviceLayout, Guard, KernelId,  # noqa: F401
                       KernelTimes, Layout, Numerics, Order, Path, SphParams, empty_particles)
from .sph import (CellGrid, Context, InitConfig, ParticleStore, build_grid, default_context,  # noqa: F401
                  drift_one, grid_nx, kick1_one, kick2_one, make_particles, run_sweep,
                  update_count)
from ._lib import SphError, load  # noqa: F401
