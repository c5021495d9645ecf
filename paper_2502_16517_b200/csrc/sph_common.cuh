// sph_common.cuh — device-side data types shared by every kernel translation unit.
//
// The 272-byte AoS record mirrors soaview::sph::Particle (reference
// include/soaview/sph/particle.hpp:11-46). The SoA mirror (`SoaMirror`) holds one
// array per field the five kernels touch (their access sets, kernels.cpp:741-859), with
// 2-vectors stored as double2 so a warp moves them with 16-byte coalesced accesses.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sphb {

struct __align__(16) Particle {
  double x[2], v[2], v_pred[2], a[2];
  double m, rho, p, u, u_pred, u_dt, c, h, wcount, rho_dh, rot_v, div_v, v_sig, h_dt, dt_next;
  int32_t frozen, moved;
  int64_t id, cell, flags;
  double dbg[2], spare[5];
};
static_assert(sizeof(Particle) == 272, "record layout must stay 272 bytes");
static_assert(offsetof(Particle, m) == 64, "particle.hpp:41");
static_assert(offsetof(Particle, frozen) == 184, "particle.hpp:42");
static_assert(offsetof(Particle, moved) == 188, "particle.hpp:43");
static_assert(offsetof(Particle, id) == 192, "particle.hpp:44");
static_assert(offsetof(Particle, dbg) == 216, "particle.hpp:45");
static_assert(offsetof(Particle, spare) == 232, "particle.hpp:46");

struct Params {
  double dt, gamma, cfl, grav, target_wcount;
};

// Field-group bits, used for dirty tracking (what sph_download must write back) and for
// the per-kernel gather/scatter views.
enum Field : uint32_t {
  F_X = 1u << 0, F_V = 1u << 1, F_VPRED = 1u << 2, F_A = 1u << 3, F_M = 1u << 4,
  F_RHO = 1u << 5, F_P = 1u << 6, F_U = 1u << 7, F_UPRED = 1u << 8, F_UDT = 1u << 9,
  F_C = 1u << 10, F_H = 1u << 11, F_WCOUNT = 1u << 12, F_RHODH = 1u << 13,
  F_ROTV = 1u << 14, F_DIVV = 1u << 15, F_VSIG = 1u << 16, F_HDT = 1u << 17,
  F_DTNEXT = 1u << 18, F_FROZEN = 1u << 19, F_MOVED = 1u << 20, F_FLAGS = 1u << 21,
  F_DBG = 1u << 22, F_CELL = 1u << 23,
  F_ALL_SOA = (1u << 24) - 1
};

// Access sets per kernel (reference view descriptors kernels.cpp:741-859).
// IN = fields read, OUT = fields written.
// flags is read-modify-write on a failed h-iteration (kernels.cpp:222), so it is InOut
constexpr uint32_t DEN_IN = F_X | F_VPRED | F_M | F_H | F_FLAGS;
constexpr uint32_t DEN_OUT = F_H | F_RHO | F_WCOUNT | F_RHODH | F_ROTV | F_DIVV | F_FLAGS;
constexpr uint32_t FOR_IN = F_X | F_VPRED | F_M | F_H | F_P | F_RHO | F_RHODH | F_C | F_DIVV |
                            F_ROTV | F_HDT;
constexpr uint32_t FOR_OUT = F_A | F_UDT | F_VSIG | F_HDT;
constexpr uint32_t DRIFT_IN = F_X | F_VPRED | F_FROZEN | F_U | F_UDT;
constexpr uint32_t DRIFT_OUT = F_X | F_UPRED | F_MOVED;
constexpr uint32_t KICK1_IN = F_V | F_A | F_U | F_UDT;
constexpr uint32_t KICK1_OUT = F_V | F_U | F_DTNEXT;
constexpr uint32_t KICK2_IN = F_V | F_A | F_DBG | F_U | F_UDT | F_UPRED | F_RHO | F_DTNEXT |
                              F_H | F_VSIG | F_C;
constexpr uint32_t KICK2_OUT = F_V | F_U | F_UPRED | F_DTNEXT | F_C | F_VPRED | F_P | F_HDT;

// Resident / scratch SoA mirror: one array per field, device slot order.
struct SoaMirror {
  double2 *x, *v, *vp, *a;
  double *m, *rho, *p, *u, *u_pred, *u_dt, *c, *h, *wcount, *rho_dh, *rot_v, *div_v, *v_sig,
      *h_dt, *dt_next, *dbg0;
  int32_t *frozen, *moved;
  int64_t *flags;
};

// Geometry of the bound grid on the device. Slots are cell-major: cell c owns slots
// [cell_begin[c], cell_begin[c+1]) in CellGrid::local order.
struct Geom {
  int nx, ny, ncells;
  int use_shift;        // 1: per-neighbour-cell periodic shift (nx,ny >= 5); 0: per-pair min image
  double cell_size;
  const int *cell_begin; // ncells + 1
};

// Deduplicated, wrapped 3x3 stencil in (dy, dx) row-major order (grid.cpp:161-176), plus
// the periodic image shift of each neighbour cell relative to cell c.
struct Stencil {
  int n;
  int cell[9];
  signed char sx[9], sy[9];
};

__host__ __device__ inline Stencil make_stencil(int c, int nx, int ny) {
  Stencil s;
  s.n = 0;
  int cy = c / nx, cx = c - cy * nx;
  for (int dy = -1; dy <= 1; ++dy)
    for (int dx = -1; dx <= 1; ++dx) {
      int wy = (cy + dy + ny) % ny, wx = (cx + dx + nx) % nx, ci = wy * nx + wx;
      bool seen = false;
      for (int k = 0; k < s.n; ++k) seen |= (s.cell[k] == ci);
      if (!seen) {
        s.cell[s.n] = ci;
        s.sx[s.n] = (signed char)(cx + dx < 0 ? -1 : (cx + dx >= nx ? 1 : 0));
        s.sy[s.n] = (signed char)(cy + dy < 0 ? -1 : (cy + dy >= ny ? 1 : 0));
        ++s.n;
      }
    }
  return s;
}

// Pair-kernel work item: `count` local particles of `cell`, whose slots are
// list[start .. start+count).
struct Item {
  int cell, start, count, pad;
};

constexpr double kSupport = 2.5;                   // spline.hpp:8
constexpr double kNorm2d = 0.025486029252413597;   // spline.hpp:9

} // namespace sphb
