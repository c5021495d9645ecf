// pair_kernels.cuh — the density and force neighbour sweeps (reference kernels.cpp:97-303,
// :535-628), as one CUDA skeleton parameterised by a numerics policy.
//
// Work decomposition (replaces the std::thread cell pool, kernels.cpp:492-533):
//   * one WARP per work item = (cell c, up to 32 local particles of c), one lane per local
//     particle i. Each lane accumulates its sums in registers over the whole active list of
//     c in the reference's order (stencil cells in (dy,dx) order, each in local-list
//     order). No reduction across lanes and no atomics on the sums, so the EXACT policy
//     reproduces the reference's summation order bit for bit.
//   * the active list streams through a per-warp shared-memory tile of 32 particles: lane
//     l gathers active particle (32k + l) — the on-the-fly AoS->SoA conversion, from the
//     AoS record or the SoA mirror — with the per-j invariants (grav*m, p/rho^2, m/rho)
//     hoisted into the tile. The next tile's global loads are in flight in registers while
//     the current tile is consumed; every lane then reads the same j (smem broadcast).
//     Warps never wait for each other (only __syncwarp), so divergence in one warp does
//     not stall its neighbours at a CTA barrier.
//   * the last tile is padded with inert dummies (x = 1e30, m = 0): every policy provably
//     skips them, so tiles always hold 32 entries and the j loop has a fixed trip count.
//   * the local particles of a cell are assigned to lanes in a spatially sorted order
//     (ilist: 8x8 sub-cell Morton bins), so the 32 lanes of a warp are neighbours and take
//     the in-support branch together; the assignment does not affect any result.
//   * density's smoothing-length iteration (kernels.cpp:184-192) runs as rounds: lanes that
//     need another round raise a flag; an order-preserving per-cell compaction builds the
//     next round's list (still in spatial order, so warps stay coherent) and the next launch
//     processes only those particles, regrouped into full warps by cell.
#pragma once
#include "sph_common.cuh"

namespace sphb {

constexpr int kTI = 32;        // local particles per work item (one warp)
constexpr int kTJ = 32;        // active particles per shared-memory tile
constexpr int kWarpsPerCta = 4;
constexpr double kDummyX = 1.0e30;
#ifndef SPH_FJ
#define SPH_FJ 2 // force: pairs per interleaved gravity group
#endif
// min resident CTAs per SM requested from ptxas (caps registers: 65536 / (128 * MINB))
#ifndef SPH_MINB_DEN
#define SPH_MINB_DEN 5
#endif
#ifndef SPH_MINB_FOR
#define SPH_MINB_FOR 5
#endif

// Per-sweep j-view (FAST numerics): the fields a pair sweep reads from its active
// particles, gathered once per sweep into SoA arrays in the spatial ilist order (index =
// cell_begin[c] + position in the cell's ilist), with the per-j invariants hoisted
// (grav*m, m*p/rho^2, m/rho). Chunk gathers are then contiguous loads with no
// indirection and no division — the paper's AoS->SoA view, built once instead of per tile.
struct JView {
  const double2 *xy, *vv; // position, v_pred
  const double *m;        // density: m
  const double2 *mg, *pv; // force: (m, grav*m), (m*p/rho^2, m/rho)
  const double *c;        // force: sound speed
};

// Issue-lean FAST density (density2_kernel, kernels_fast.cu): j-view split for vector LDS.
struct D2View {
  const double *x, *y, *m; // position, mass
  const double2 *vv;       // v_pred
};

struct DenArgs {
  Geom g;
  const Item *items;
  int n_items;
  const int *list;      // slots, indexed by Item::start
  int round;            // h-iteration round (0..29)
  double target, h_max;
  const Particle *aos;  // AoS source / destination (AOS instantiation)
  SoaMirror soa;        // SoA source / destination (SoA instantiation)
  double *hcur;         // per-slot h of the pending round
  unsigned char *again; // per list position: 1 if the particle needs another round
  unsigned char *rounds_out; // optional per-slot round count (stats / parity analysis)
  double *wc_out;       // mean_wcount mode: per-slot neighbour sum (grid.cpp:36-50)
  const int *jlist;     // culled FAST sweep: cell-major slots in spatial order (ilist)
  const float4 *boxes;  // culled FAST sweep: bounding box of each 32-chunk of jlist
  JView jv;             // culled FAST sweep: j-view in jlist order
  D2View jv2;           // issue-lean FAST sweep (resident SoA): split j-view (x null = off)
  double k0375;         // series constant (kernel parameter -> constant-bank operand)
  int jslices;          // density2: lanes per local particle (1, 2, 4); items hold 32/jslices
  unsigned long long *fail_count; // optional: particles that hit the 30-round limit
                                  // (density_step's Fail, kernels.cpp:190), for sph_stats
  int *item_ctr;          // density2: non-null = persistent launch, warps take items from it
  const int *n_items_dev; // density2 persistent launch: item count in device memory (else n_items)
};

struct ForArgs {
  Geom g;
  const Item *items;
  int n_items;
  const int *list;
  double grav;
  const Particle *aos;
  SoaMirror soa;
  const int *jlist;     // FAST: j in spatial order (ilist); null = reference order
  const float4 *boxes;  // FAST: chunk boxes -> far chunks take the gravity-only path
  JView jv;             // FAST: j-view in jlist order (null xy = gather from the mirror)
};

// Issue-lean FAST force (force2_kernel, kernels_fast.cu): j-view split for vector LDS.
// Chunk-major j-view of the force sweep: block G holds x[32], y[32], grav*m[32],
// v_pred[32], (P = m p / rho^2, V = m / rho)[32], (c, m)[32] in the tile layout (2304 bytes),
// padded with inert dummies (x = 1e30, gm = 0).
constexpr int kF2Blk = 288; // doubles per force block
struct F2View {
  const double *blk;
};

struct F2Args {
  Geom g;
  const Item *items;
  int n_items;
  const int *list;
  double grav;
  const Particle *aos;  // non-null: i side read and written in the AoS records (AOS layout)
  SoaMirror soa;
  const float4 *boxes;
  F2View jv;
  double k1875, k0375; // series constants (kernel parameters -> constant-bank operands)
  int *item_ctr;       // non-null: persistent launch, warps take items from this counter
  const int *n_items_dev; // persistent launch: the item count in device memory (else n_items)
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

// Per-warp active-list layout: stencil cells, their slot ranges and prefix offsets.
struct ActiveLayout {
  int n;          // stencil cells
  int cell[9];    // stencil cell ids
  int na;         // active particles
  int pre[10];    // prefix of counts
  int nch[10];    // prefix of 32-chunks per stencil cell
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
    L.cell[k] = st.cell[k];
    L.pre[k + 1] = L.pre[k] + (e - b);
    L.sx[k] = st.sx[k];
    L.sy[k] = st.sy[k];
  }
  L.na = L.pre[st.n];
  L.nch[0] = 0;
  for (int k = 0; k < st.n; ++k) L.nch[k + 1] = L.nch[k] + (L.pre[k + 1] - L.pre[k] + 31) / 32;
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

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_in_cta() { return threadIdx.x >> 5; }

// ---------------------------------------------------------------------------------------
// Density round (also the mean_wcount pass of make_particles when MEANW).
// ---------------------------------------------------------------------------------------
template <class P, bool AOS, bool MEANW>
__global__ void __launch_bounds__(kWarpsPerCta * 32, SPH_MINB_DEN) density_round_kernel(DenArgs A) {
  __shared__ DenTile tiles[kWarpsPerCta];
  __shared__ ActiveLayout lay[kWarpsPerCta];
  const int w = warp_in_cta(), lane = lane_id();
  const int item_idx = blockIdx.x * kWarpsPerCta + w;
  if (item_idx >= A.n_items) return; // whole warp
  DenTile &T = tiles[w];
  ActiveLayout &L = lay[w];
  const Item it = A.items[item_idx];
  if (lane == 0) build_active(A.g, it.cell, L);
  JSrc<AOS> src;
  if constexpr (AOS) src.p = A.aos; else src.f = A.soa;
  const bool live = lane < it.count;
  const int slot = A.list[it.start + (live ? lane : 0)];
  const double2 xi = src.x(slot), vi = src.vp(slot);
  const double mi = src.m(slot);
  const double h = (A.round == 0) ? src.h(slot) : A.hcur[slot];
  __syncwarp();
  const bool minimg = P::kExactOrder || !A.g.use_shift;
  const int na = L.na, ntiles = (na + kTJ - 1) / kTJ;

  typename P::DI I = P::den_i(xi.x, xi.y, vi.x, vi.y, h);
  typename P::DA s = P::den_zero();
  typename P::MW mw = P::mw_zero();

  double2 rx, rv;
  double rm;
  auto gather = [&](int k) {
    const int p = k * kTJ + lane;
    if (p < na) {
      int nb;
      const int sj = active_slot(L, p, nb);
      rx = src.x(sj);
      rv = src.vp(sj);
      rm = src.m(sj);
      if (!minimg) { rx.x += L.sx[nb]; rx.y += L.sy[nb]; }
    } else { // inert padding (skipped by every policy)
      rx = make_double2(kDummyX, kDummyX);
      rv = make_double2(0.0, 0.0);
      rm = 0.0;
    }
  };
  if (ntiles > 0) gather(0);
  for (int k = 0; k < ntiles; ++k) {
    T.xy[lane] = rx;
    T.vv[lane] = rv;
    T.m[lane] = rm;
    __syncwarp();
    if (k + 1 < ntiles) gather(k + 1); // loads in flight during the tile
    if (MEANW) {
      if (minimg) P::template mw_tile<true>(I, T, mw);
      else P::template mw_tile<false>(I, T, mw);
    } else {
      if (minimg) P::template den_tile<true>(I, T, s);
      else P::template den_tile<false>(I, T, s);
    }
    __syncwarp();
  }
  if (!live) return;
  if (MEANW) {
    A.wc_out[slot] = P::mw_value(mw);
    return;
  }
  double hn = h;
  const int st = P::den_step(s, hn, A.target, A.h_max, A.round);
  A.again[it.start + lane] = (unsigned char)(st == 0);
  if (st == 0) { // Again: next round with hn (list compacted in order by compact_pending)
    A.hcur[slot] = hn;
    return;
  }
  double o[6]; // h, rho, wcount, rho_dh, rot_v, div_v
  P::den_publish(s, h, mi, o);
  if (A.rounds_out) A.rounds_out[slot] = (unsigned char)(A.round + 1);
  if (st == 2 && A.fail_count) atomicAdd(A.fail_count, 1ull);
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

__device__ __forceinline__ int chunk_box_index(int cell_begin_c, int c, int k) {
  return (cell_begin_c >> 5) + c + k;
}

__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Chunk g of the active list -> (stencil cell nb, chunk k within it).
__device__ __forceinline__ void chunk_locate(const ActiveLayout &L, int g, int &nb, int &k) {
  nb = 0;
#pragma unroll 1
  while (nb + 1 < L.n && g >= L.nch[nb + 1]) ++nb;
  k = g - L.nch[nb];
}

// Warp box (or a single point) against the FP32 box of chunk (nb, k), shifted to the
// periodic image of stencil cell nb: true if some pair can be within `reach`.
// The near/far classification in FP32, with every rounding explicit (no contraction left to
// the compiler): the same item then classifies its chunks identically in every inlined copy
// of a sweep (persistent or one CTA per item), so FAST results do not depend on scheduling.
// reach = 2.5 max(h) (1 + 1e-5) + 1e-6 covers the FP32 rounding of the positions and boxes.
__device__ __forceinline__ float reach_of(float r25) { return __fmaf_rn(r25, 1.0f + 1e-5f, 1e-6f); }
__device__ __forceinline__ float box_gap2(float gx, float gy) {
  return __fmaf_rn(gx, gx, __fmul_rn(gy, gy));
}
__device__ __forceinline__ bool chunk_near(const ActiveLayout &L, const float4 *boxes, int nb, int k,
                                           float xlo, float xhi, float ylo, float yhi,
                                           float reach2) {
  const float4 b = boxes[chunk_box_index(L.base[nb], L.cell[nb], k)];
  const float sx = (float)L.sx[nb], sy = (float)L.sy[nb];
  const float gx = fmaxf(0.0f, fmaxf(b.x + sx - xhi, xlo - (b.z + sx)));
  const float gy = fmaxf(0.0f, fmaxf(b.y + sy - yhi, ylo - (b.w + sy)));
  return box_gap2(gx, gy) <= reach2;
}

// Visits the chunks of the active list in order, 32 at a time: lane l evaluates chunk
// g0 + l (box test, all lanes in parallel), a ballot gives the batch's chunk set, and the
// chunks are handed to `visit(nb, k, near, next_nb, next_k, has_next)` in order so the
// caller can prefetch the next chunk. ALL_CHUNKS: every chunk is visited (near = box test);
// otherwise only near chunks are.
template <bool ALL_CHUNKS, class Visit>
__device__ __forceinline__ void walk_chunks(const ActiveLayout &L, const float4 *boxes, bool test,
                                            float xlo, float xhi, float ylo, float yhi,
                                            float reach2, Visit &&visit) {
  const int lane = threadIdx.x & 31;
  const int total = L.nch[L.n];
  for (int g0 = 0; g0 < total; g0 += 32) {
    const int g = g0 + lane;
    int nb = 0, k = 0;
    bool valid = g < total, near = valid;
    if (valid) {
      chunk_locate(L, g, nb, k);
      if (test) near = chunk_near(L, boxes, nb, k, xlo, xhi, ylo, yhi, reach2);
    }
    const unsigned vmask = __ballot_sync(0xffffffffu, valid);
    const unsigned nmask = __ballot_sync(0xffffffffu, near);
    unsigned todo = ALL_CHUNKS ? vmask : nmask;
    while (todo) {
      const int b = __ffs(todo) - 1;
      todo &= todo - 1;
      const int bn = todo ? __ffs(todo) - 1 : 0;
      const int cnb = __shfl_sync(0xffffffffu, nb, b), ck = __shfl_sync(0xffffffffu, k, b);
      const int nnb = __shfl_sync(0xffffffffu, nb, bn), nk = __shfl_sync(0xffffffffu, k, bn);
      visit(cnb, ck, ((nmask >> b) & 1u) != 0u, nnb, nk, todo != 0u);
    }
  }
}

// ---------------------------------------------------------------------------------------
// Force sweep. The active list is walked per stencil cell in 32-particle chunks (chunk
// prefix kept in shared memory, so no per-lane search); the next chunk's loads are in
// flight while the current one is consumed. With FAST numerics the chunks follow the
// spatial ilist order and a chunk farther than the warp's support reach from the warp's
// bounding box takes the gravity-only path (the softened gravity acts on every active
// pair, kernels.cpp:128-131, but no SPH term can be in support there).
// ---------------------------------------------------------------------------------------
template <class P, bool AOS, bool VIEW>
__global__ void __launch_bounds__(kWarpsPerCta * 32, SPH_MINB_FOR) force_kernel(ForArgs A) {
  __shared__ ForTile tiles[kWarpsPerCta];
  __shared__ ActiveLayout lay[kWarpsPerCta];
  __shared__ typename P::FCold cold[kWarpsPerCta * 32];
  const int w = warp_in_cta(), lane = lane_id();
  const int item_idx = blockIdx.x * kWarpsPerCta + w;
  if (item_idx >= A.n_items) return;
  ForTile &T = tiles[w];
  ActiveLayout &L = lay[w];
  const Item it = A.items[item_idx];
  if (lane == 0) build_active(A.g, it.cell, L);
  JSrc<AOS> src;
  if constexpr (AOS) src.p = A.aos; else src.f = A.soa;
  const bool live = lane < it.count;
  const int slot = A.list[it.start + (live ? lane : 0)];
  const double2 xi = src.x(slot);
  const double hi = src.h(slot);
  typename P::FI I = P::for_i(xi, src.vp(slot), hi, src.pr(slot), src.rho(slot),
                              src.rho_dh(slot), src.c(slot), src.div_v(slot), src.rot_v(slot),
                              A.grav, &cold[threadIdx.x]);
  typename P::FA s = P::for_zero(src.h_dt(slot));
  const bool cull = A.boxes != nullptr;
  float ixlo = 0.f, ixhi = 0.f, iylo = 0.f, iyhi = 0.f, reach2 = 0.f;
  if (cull) {
    ixlo = warp_min((float)xi.x);
    ixhi = warp_max((float)xi.x);
    iylo = warp_min((float)xi.y);
    iyhi = warp_max((float)xi.y);
    const float reach = reach_of(warp_max((float)(2.5 * hi)));
    reach2 = __fmul_rn(reach, reach);
  }
  __syncwarp();
  const bool minimg = P::kExactOrder || !A.g.use_shift;

  double2 rx, rv, rmg, rpv;
  double rm, rrho, rp, rc;
  auto gather = [&](int nb, int k) {
    const int cnt = L.pre[nb + 1] - L.pre[nb];
    const int q = k * kTJ + lane;
    if (q < cnt) {
      const int idx = L.base[nb] + q;
      if constexpr (VIEW) { // contiguous j-view loads, derived terms precomputed
        rx = A.jv.xy[idx];
        rv = A.jv.vv[idx];
        rmg = A.jv.mg[idx];
        rpv = A.jv.pv[idx];
        rc = A.jv.c[idx];
      } else {
        const int sj = A.jlist ? A.jlist[idx] : idx;
        rx = src.x(sj);
        rv = src.vp(sj);
        rm = src.m(sj);
        rrho = src.rho(sj);
        rp = src.pr(sj);
        rc = src.c(sj);
      }
    } else { // inert padding: r2 <= 0 (exact) or gm = 0 (fast)
      rx = make_double2(kDummyX, kDummyX);
      rv = make_double2(0.0, 0.0);
      rm = 0.0; rrho = 1.0; rp = 0.0; rc = 0.0;
      rmg = make_double2(0.0, 0.0);
      rpv = make_double2(0.0, 0.0);
    }
  };
  bool staged = false; // registers already hold the chunk about to be consumed
  int gnb = 0;          // stencil cell of the staged chunk (periodic shift applied at staging)
  walk_chunks<true>(L, A.boxes, cull && !minimg, ixlo, ixhi, iylo, iyhi, reach2,
                    [&](int nb, int k, bool near, int nnb, int nk, bool has_next) {
    if (!staged) { gather(nb, k); gnb = nb; }
    double2 sxy = rx;
    if (!minimg) { sxy.x += L.sx[gnb]; sxy.y += L.sy[gnb]; }
    T.xy[lane] = sxy;
    T.vv[lane] = rv;
    if constexpr (VIEW) {
      T.mg[lane] = rmg;
      T.pv[lane] = rpv;
    } else {
      const double4 d = P::stage_force(rm, rrho, rp, A.grav); // (m, gm, pv.x, pv.y)
      T.mg[lane] = make_double2(d.x, d.y);
      T.pv[lane] = make_double2(d.z, d.w);
    }
    T.c[lane] = rc;
    __syncwarp();
    staged = has_next;
    if (has_next) { gather(nnb, nk); gnb = nnb; } // loads in flight during this chunk
    if (minimg) P::template for_tile<true>(I, T, s);
    else if (near) P::template for_tile<false>(I, T, s);
    else P::template for_tile_far(I, T, s);
    __syncwarp();
  });
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

// ---------------------------------------------------------------------------------------
// Culled density round (FAST numerics only; the j order is the spatial ilist order, which
// the EXACT policy cannot use). The active list is walked per stencil cell in 32-particle
// chunks of ilist; a chunk whose bounding box (precomputed, chunk_box_kernel) lies farther
// than the warp's largest support radius 2.5 max(h_i) from the warp's own bounding box holds
// no in-support pair for any lane (|x_i - x_j| < 2.5 h_i is necessary) and is skipped
// without being loaded. Boxes are in FP32 with an absolute safety margin of 1e-6.
// Chunk k of cell c has box index (cell_begin[c] >> 5) + c + k (unique, no scan needed).
// ---------------------------------------------------------------------------------------
template <class P, bool AOS>
__global__ void __launch_bounds__(kWarpsPerCta * 32, SPH_MINB_DEN) density_cull_kernel(DenArgs A) {
  __shared__ DenTile tiles[kWarpsPerCta];
  __shared__ ActiveLayout lay[kWarpsPerCta];
  const int w = warp_in_cta(), lane = lane_id();
  const int item_idx = blockIdx.x * kWarpsPerCta + w;
  if (item_idx >= A.n_items) return;
  DenTile &T = tiles[w];
  ActiveLayout &L = lay[w];
  const Item it = A.items[item_idx];
  if (lane == 0) build_active(A.g, it.cell, L);
  JSrc<AOS> src;
  if constexpr (AOS) src.p = A.aos; else src.f = A.soa;
  const bool live = lane < it.count;
  const int slot = A.list[it.start + (live ? lane : 0)];
  const double2 xi = src.x(slot), vi = src.vp(slot);
  const double mi = src.m(slot);
  const double h = (A.round == 0) ? src.h(slot) : A.hcur[slot];
  typename P::DI I = P::den_i(xi.x, xi.y, vi.x, vi.y, h);
  typename P::DA s = P::den_zero();
  // warp bounding box and reach (dead lanes carry lane 0's particle)
  const float ixlo = warp_min((float)xi.x), ixhi = warp_max((float)xi.x);
  const float iylo = warp_min((float)xi.y), iyhi = warp_max((float)xi.y);
  const float reach = reach_of(warp_max((float)(2.5 * h)));
  const float reach2 = __fmul_rn(reach, reach);
  __syncwarp();
  const bool minimg = !A.g.use_shift;
  double2 rx, rv;
  double rm;
  auto gather = [&](int nb, int k) {
    const int cnt = L.pre[nb + 1] - L.pre[nb];
    const int q = k * kTJ + lane;
    if (q < cnt) {
      const int idx = L.base[nb] + q;
      if (A.jv.xy) {
        rx = A.jv.xy[idx];
        rv = A.jv.vv[idx];
        rm = A.jv.m[idx];
      } else {
        const int sj = A.jlist[idx];
        rx = src.x(sj);
        rv = src.vp(sj);
        rm = src.m(sj);
      }
    } else {
      rx = make_double2(kDummyX, kDummyX);
      rv = make_double2(0.0, 0.0);
      rm = 0.0;
    }
  };
  bool staged = false;
  int gnb = 0;
  walk_chunks<false>(L, A.boxes, !minimg, ixlo, ixhi, iylo, iyhi, reach2,
                     [&](int nb, int k, bool, int nnb, int nk, bool has_next) {
    if (!staged) { gather(nb, k); gnb = nb; }
    double2 sxy = rx;
    if (!minimg) { sxy.x += L.sx[gnb]; sxy.y += L.sy[gnb]; }
    T.xy[lane] = sxy;
    T.vv[lane] = rv;
    T.m[lane] = rm;
    __syncwarp();
    staged = has_next;
    if (has_next) { gather(nnb, nk); gnb = nnb; }
    if (minimg) P::template den_tile<true>(I, T, s);
    else P::template den_tile<false>(I, T, s);
    __syncwarp();
  });
  if (!live) return;
  double hn = h;
  const int st = P::den_step(s, hn, A.target, A.h_max, A.round);
  A.again[it.start + lane] = (unsigned char)(st == 0);
  if (st == 0) {
    A.hcur[slot] = hn;
    return;
  }
  double o[6];
  P::den_publish(s, h, mi, o);
  if (A.rounds_out) A.rounds_out[slot] = (unsigned char)(A.round + 1);
  if (st == 2 && A.fail_count) atomicAdd(A.fail_count, 1ull);
  if constexpr (AOS) {
    Particle &pq = const_cast<Particle &>(A.aos[slot]);
    pq.h = o[0]; pq.rho = o[1]; pq.wcount = o[2]; pq.rho_dh = o[3]; pq.rot_v = o[4]; pq.div_v = o[5];
    if (st == 2) pq.flags += 1;
  } else {
    A.soa.h[slot] = o[0]; A.soa.rho[slot] = o[1]; A.soa.wcount[slot] = o[2];
    A.soa.rho_dh[slot] = o[3]; A.soa.rot_v[slot] = o[4]; A.soa.div_v[slot] = o[5];
    if (st == 2) A.soa.flags[slot] += 1;
  }
}

inline int pair_grid(int n_items) { return (n_items + kWarpsPerCta - 1) / kWarpsPerCta; }

} // namespace sphb
