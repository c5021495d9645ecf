// pair_kernels.cuh — the density and force neighbour sweeps (reference kernels.cpp:97-303,
// :535-628), as one CUDA skeleton parameterised by a numerics policy.
//
// Work decomposition (replaces the std::thread cell pool, kernels.cpp:492-533):
//   * one CTA per work item = (cell c, up to kTI local particles of c); one thread per
//     local particle i, which accumulates its sums in registers over the whole active list
//     of c in the reference's order (stencil cells in (dy,dx) order, each in local-list
//     order). There is no reduction across threads and no atomics on the sums, so the
//     EXACT policy reproduces the reference's summation order bit for bit.
//   * the active list streams through shared memory in tiles of kTJ particles: every
//     thread gathers one j record (AoS record or SoA mirror -> SoA tile: the on-the-fly
//     AoS->SoA conversion), per-j invariants (grav*m, p/rho^2, m/rho) are hoisted into the
//     tile, and the tile is double-buffered (global loads for tile k+1 are in flight while
//     tile k is consumed). All lanes of a warp read the same j (shared-memory broadcast).
//   * the local particles of a cell are assigned to threads in a spatially sorted order
//     (ilist), so the 32 lanes of a warp are neighbours and take the in-support branch
//     together; the assignment does not affect any particle's result.
//   * density's smoothing-length iteration (kernels.cpp:184-192) runs as rounds: particles
//     that need another round append themselves to a per-cell pending list and the next
//     launch only processes those (grouped by cell again), instead of re-sweeping tiles.
#pragma once
#include "sph_common.cuh"

namespace sphb {

constexpr int kTI = 128; // local particles (threads) per CTA
constexpr int kTJ = 128; // active particles per shared-memory tile

struct DenArgs {
  Geom g;
  const Item *items;
  const int *list;      // slots, indexed by Item::start
  int round;            // h-iteration round (0..29)
  double target, h_max;
  const Particle *aos;  // AoS source / destination (AOS instantiation)
  SoaMirror soa;        // SoA source / destination (SoA instantiation)
  double *hcur;         // per-slot h of the pending round
  int *pend_cnt;        // per-cell pending counters (next round)
  int *pend_list;       // next-round slots, cell c at [cell_begin[c], ...)
  unsigned char *rounds_out; // optional per-slot round count (stats / parity analysis)
  double *wc_out;       // mean_wcount mode: per-slot neighbour sum (grid.cpp:36-50)
};

struct ForArgs {
  Geom g;
  const Item *items;
  const int *list;
  double grav;
  const Particle *aos;
  SoaMirror soa;
};

// ---- j staging (gather one active record into the SoA tile) ----
template <bool AOS> struct JSrc;
template <> struct JSrc<true> {
  const Particle *p;
  __device__ __forceinline__ double2 x(int s) const { return *reinterpret_cast<const double2 *>(p[s].x); }
  __device__ __forceinline__ double2 vp(int s) const { return *reinterpret_cast<const double2 *>(p[s].v_pred); }
  __device__ __forceinline__ double m(int s) const { return p[s].m; }
  __device__ __forceinline__ double rho(int s) const { return p[s].rho; }
  __device__ __forceinline__ double pr(int s) const { return p[s].p; }
  __device__ __forceinline__ double c(int s) const { return p[s].c; }
  __device__ __forceinline__ double h(int s) const { return p[s].h; }
  __device__ __forceinline__ double rho_dh(int s) const { return p[s].rho_dh; }
  __device__ __forceinline__ double div_v(int s) const { return p[s].div_v; }
  __device__ __forceinline__ double rot_v(int s) const { return p[s].rot_v; }
  __device__ __forceinline__ double h_dt(int s) const { return p[s].h_dt; }
};
template <> struct JSrc<false> {
  SoaMirror f;
  __device__ __forceinline__ double2 x(int s) const { return f.x[s]; }
  __device__ __forceinline__ double2 vp(int s) const { return f.vp[s]; }
  __device__ __forceinline__ double m(int s) const { return f.m[s]; }
  __device__ __forceinline__ double rho(int s) const { return f.rho[s]; }
  __device__ __forceinline__ double pr(int s) const { return f.p[s]; }
  __device__ __forceinline__ double c(int s) const { return f.c[s]; }
  __device__ __forceinline__ double h(int s) const { return f.h[s]; }
  __device__ __forceinline__ double rho_dh(int s) const { return f.rho_dh[s]; }
  __device__ __forceinline__ double div_v(int s) const { return f.div_v[s]; }
  __device__ __forceinline__ double rot_v(int s) const { return f.rot_v[s]; }
  __device__ __forceinline__ double h_dt(int s) const { return f.h_dt[s]; }
};

// Per-CTA active-list layout: stencil cells, their slot ranges and prefix offsets.
struct ActiveLayout {
  int n;          // stencil cells
  int na;         // active particles
  int pre[10];    // prefix of counts
  int base[9];    // first slot of each stencil cell
  double sx[9], sy[9]; // periodic image shift of each stencil cell
};

__device__ __forceinline__ void build_active(const Geom &g, int c, ActiveLayout &L) {
  Stencil st = make_stencil(c, g.nx, g.ny);
  L.n = st.n;
  L.pre[0] = 0;
  for (int k = 0; k < st.n; ++k) {
    int b = g.cell_begin[st.cell[k]], e = g.cell_begin[st.cell[k] + 1];
    L.base[k] = b;
    L.pre[k + 1] = L.pre[k] + (e - b);
    L.sx[k] = st.sx[k];
    L.sy[k] = st.sy[k];
  }
  L.na = L.pre[st.n];
}

// Active position p -> (slot, stencil index).
__device__ __forceinline__ int active_slot(const ActiveLayout &L, int p, int &k) {
  k = 0;
#pragma unroll 1
  while (k + 1 < L.n && p >= L.pre[k + 1]) ++k;
  return L.base[k] + (p - L.pre[k]);
}

struct DenTile {
  double2 xy[kTJ];
  double2 vv[kTJ];
  double m[kTJ];
};

struct ForTile {
  double2 xy[kTJ];
  double2 vv[kTJ];
  double2 mg[kTJ]; // (m, grav*m)
  double2 pv[kTJ]; // policy-defined pressure / volume terms
  double c[kTJ];
};

// ---------------------------------------------------------------------------------------
// Density round (also the mean_wcount pass of make_particles when MEANW).
// ---------------------------------------------------------------------------------------
template <class P, bool AOS, bool MEANW>
__global__ void __launch_bounds__(kTI) density_round_kernel(DenArgs A) {
  __shared__ DenTile tile[2];
  __shared__ ActiveLayout L;
  const Item it = A.items[blockIdx.x];
  const int t = threadIdx.x;
  if (t == 0) build_active(A.g, it.cell, L);
  JSrc<AOS> src;
  if constexpr (AOS) src.p = A.aos; else src.f = A.soa;
  const bool live = t < it.count;
  const bool warp_live = (t & ~31) < it.count;
  const int slot = A.list[it.start + (live ? t : 0)];
  const double2 xi = src.x(slot), vi = src.vp(slot);
  const double mi = src.m(slot);
  double h = (A.round == 0) ? src.h(slot) : A.hcur[slot];
  __syncthreads();
  const bool minimg = P::kExactOrder || !A.g.use_shift;
  const int na = L.na, ntiles = (na + kTJ - 1) / kTJ;

  typename P::DI I = P::den_i(xi.x, xi.y, vi.x, vi.y, h);
  typename P::DA s = P::den_zero();
  typename P::MW mw = P::mw_zero();

  // prologue: gather tile 0
  double2 rx = make_double2(0.0, 0.0), rv = rx;
  double rm = 0.0;
  auto gather = [&](int k) {
    int p = k * kTJ + t;
    if (p < na) {
      int nb;
      int sj = active_slot(L, p, nb);
      rx = src.x(sj);
      rv = src.vp(sj);
      rm = src.m(sj);
      if (!minimg) { rx.x += L.sx[nb]; rx.y += L.sy[nb]; }
    }
  };
  auto store = [&](DenTile &T) {
    T.xy[t] = rx;
    T.vv[t] = rv;
    T.m[t] = rm;
  };
  if (ntiles > 0) {
    gather(0);
    store(tile[0]);
  }
  __syncthreads();
  for (int k = 0; k < ntiles; ++k) {
    if (k + 1 < ntiles) gather(k + 1);
    const DenTile &T = tile[k & 1];
    const int tn = min(kTJ, na - k * kTJ);
    if (warp_live) {
      if (MEANW) {
        if (minimg) {
#pragma unroll 4
          for (int j = 0; j < tn; ++j) P::template mw_pair<true>(I, T.xy[j], mw);
        } else {
#pragma unroll 4
          for (int j = 0; j < tn; ++j) P::template mw_pair<false>(I, T.xy[j], mw);
        }
      } else if (minimg) {
#pragma unroll 4
        for (int j = 0; j < tn; ++j) P::template den_pair<true>(I, T.xy[j], T.vv[j], T.m[j], s);
      } else {
#pragma unroll 4
        for (int j = 0; j < tn; ++j) P::template den_pair<false>(I, T.xy[j], T.vv[j], T.m[j], s);
      }
    }
    if (k + 1 < ntiles) store(tile[(k + 1) & 1]);
    __syncthreads();
  }
  if (!live) return;
  if (MEANW) {
    A.wc_out[slot] = P::mw_value(mw);
    return;
  }
  double hn = h;
  const int st = P::den_step(s, hn, A.target, A.h_max, A.round);
  if (st == 0) { // Again: next round with hn
    A.hcur[slot] = hn;
    const int pos = atomicAdd(&A.pend_cnt[it.cell], 1);
    A.pend_list[A.g.cell_begin[it.cell] + pos] = slot;
    return;
  }
  double o[6]; // h, rho, wcount, rho_dh, rot_v, div_v
  P::den_publish(s, h, mi, o);
  if (A.rounds_out) A.rounds_out[slot] = (unsigned char)(A.round + 1);
  if constexpr (AOS) {
    Particle &q = const_cast<Particle &>(A.aos[slot]);
    q.h = o[0]; q.rho = o[1]; q.wcount = o[2]; q.rho_dh = o[3]; q.rot_v = o[4]; q.div_v = o[5];
    if (st == 2) q.flags += 1;
  } else {
    A.soa.h[slot] = o[0]; A.soa.rho[slot] = o[1]; A.soa.wcount[slot] = o[2];
    A.soa.rho_dh[slot] = o[3]; A.soa.rot_v[slot] = o[4]; A.soa.div_v[slot] = o[5];
    if (st == 2) A.soa.flags[slot] += 1;
  }
}

// ---------------------------------------------------------------------------------------
// Force sweep.
// ---------------------------------------------------------------------------------------
template <class P, bool AOS>
__global__ void __launch_bounds__(kTI) force_kernel(ForArgs A) {
  __shared__ ForTile tile[2];
  __shared__ ActiveLayout L;
  const Item it = A.items[blockIdx.x];
  const int t = threadIdx.x;
  if (t == 0) build_active(A.g, it.cell, L);
  JSrc<AOS> src;
  if constexpr (AOS) src.p = A.aos; else src.f = A.soa;
  const bool live = t < it.count;
  const bool warp_live = (t & ~31) < it.count;
  const int slot = A.list[it.start + (live ? t : 0)];
  typename P::FI I = P::for_i(src.x(slot), src.vp(slot), src.h(slot), src.pr(slot),
                              src.rho(slot), src.rho_dh(slot), src.c(slot), src.div_v(slot),
                              src.rot_v(slot), A.grav);
  typename P::FA s = P::for_zero(src.h_dt(slot));
  __syncthreads();
  const bool minimg = P::kExactOrder || !A.g.use_shift;
  const int na = L.na, ntiles = (na + kTJ - 1) / kTJ;

  double2 rx = make_double2(0.0, 0.0), rv = rx;
  double rm = 0.0, rrho = 1.0, rp = 0.0, rc = 0.0;
  auto gather = [&](int k) {
    int p = k * kTJ + t;
    if (p < na) {
      int nb;
      int sj = active_slot(L, p, nb);
      rx = src.x(sj);
      rv = src.vp(sj);
      rm = src.m(sj);
      rrho = src.rho(sj);
      rp = src.pr(sj);
      rc = src.c(sj);
      if (!minimg) { rx.x += L.sx[nb]; rx.y += L.sy[nb]; }
    }
  };
  auto store = [&](ForTile &T) {
    T.xy[t] = rx;
    T.vv[t] = rv;
    double4 d = P::stage_force(rm, rrho, rp, A.grav); // (m, gm, pv.x, pv.y)
    T.mg[t] = make_double2(d.x, d.y);
    T.pv[t] = make_double2(d.z, d.w);
    T.c[t] = rc;
  };
  if (ntiles > 0) {
    gather(0);
    store(tile[0]);
  }
  __syncthreads();
  for (int k = 0; k < ntiles; ++k) {
    if (k + 1 < ntiles) gather(k + 1);
    const ForTile &T = tile[k & 1];
    const int tn = min(kTJ, na - k * kTJ);
    if (warp_live) {
      if (minimg) {
#pragma unroll 2
        for (int j = 0; j < tn; ++j)
          P::template for_pair<true>(I, T.xy[j], T.vv[j], T.mg[j], T.pv[j], T.c[j], s);
      } else {
#pragma unroll 2
        for (int j = 0; j < tn; ++j)
          P::template for_pair<false>(I, T.xy[j], T.vv[j], T.mg[j], T.pv[j], T.c[j], s);
      }
    }
    if (k + 1 < ntiles) store(tile[(k + 1) & 1]);
    __syncthreads();
  }
  if (!live) return;
  double o[5]; // a0, a1, u_dt, v_sig, h_dt
  P::for_publish(I, s, o);
  if constexpr (AOS) {
    Particle &q = const_cast<Particle &>(A.aos[slot]);
    q.a[0] = o[0]; q.a[1] = o[1]; q.u_dt = o[2]; q.v_sig = o[3]; q.h_dt = o[4];
  } else {
    A.soa.a[slot] = make_double2(o[0], o[1]);
    A.soa.u_dt[slot] = o[2]; A.soa.v_sig[slot] = o[3]; A.soa.h_dt[slot] = o[4];
  }
}

// Host-side launchers (defined in kernels_exact.cu / kernels_fast.cu).
void launch_density_exact(const DenArgs &a, int n_items, bool aos, bool meanw, cudaStream_t s);
void launch_force_exact(const ForArgs &a, int n_items, bool aos, cudaStream_t s);
void launch_density_fast(const DenArgs &a, int n_items, bool aos, cudaStream_t s);
void launch_force_fast(const ForArgs &a, int n_items, bool aos, cudaStream_t s);

} // namespace sphb
