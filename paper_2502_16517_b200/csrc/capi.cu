// capi.cu — host runtime behind the C-ABI (include/sph_b200.h).
//
// Owns the device mirror of a bound CellGrid and drives the kernels. This replaces, in
// order: the caller-side particle container traffic of run_sweep (the reference mutates
// records through Particle* lists, kernels.cpp:861-872), the per-cell scheduler
// (sweep_cells, kernels.cpp:492-533) with a GPU work list, the per-call SoA arenas
// (layout.cpp) with resident device buffers, and build_grid (grid.cpp:145-184) with a
// device rebin. make_particles (grid.cpp:76-143) runs its sweeps on the device with the
// EXACT policy so the IC is byte-identical to the reference's.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "../../include/sph_b200.h"
#include "pair_kernels.cuh"
#include "sph_kernels.h"

using namespace sphb;

namespace {

struct CudaError {
  cudaError_t e;
  const char *what;
  int line;
};

#define CK(call)                                                                           \
  do {                                                                                     \
    cudaError_t _e = (call);                                                               \
    if (_e != cudaSuccess) throw CudaError{_e, #call, __LINE__};                          \
  } while (0)

struct ArgError {
  std::string msg;
};

template <class T> struct DevBuf {
  T *p = nullptr;
  size_t cap = 0; // elements
  void ensure(size_t n) {
    if (n <= cap && p) return;
    if (p) CK(cudaFree(p));
    p = nullptr;
    cap = 0;
    CK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    cap = std::max<size_t>(n, 1);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  // capacity for `need` elements keeping the first `keep` (25 % headroom on growth)
  void reserve_keep(size_t need, size_t keep, cudaStream_t st) {
    if (need <= cap && p) return;
    const size_t nc = std::max<size_t>(need + need / 4, 1);
    T *q = nullptr;
    CK(cudaMalloc(&q, nc * sizeof(T)));
    if (p && keep) CK(cudaMemcpyAsync(q, p, std::min(keep, cap) * sizeof(T), cudaMemcpyDeviceToDevice, st));
    if (p) {
      CK(cudaStreamSynchronize(st));
      CK(cudaFree(p));
    }
    p = q;
    cap = nc;
  }
};

struct PinnedBuf {
  void *p = nullptr;
  size_t cap = 0;
  void ensure(size_t bytes) {
    if (bytes <= cap && p) return;
    if (p) CK(cudaFreeHost(p));
    p = nullptr;
    cap = 0;
    CK(cudaMallocHost(&p, std::max<size_t>(bytes, 64)));
    cap = std::max<size_t>(bytes, 64);
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
  }
};

// Host-side parallel loop (gathers/scatters between Particle* lists and pinned staging).
template <class F> void parallel_for(int64_t n, F &&fn) {
  int nt = (int)std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()), 32);
  if (n < 65536 || nt <= 1) {
    fn((int64_t)0, n);
    return;
  }
  std::vector<std::thread> th;
  int64_t chunk = (n + nt - 1) / nt;
  for (int t = 0; t < nt; ++t) {
    int64_t b = t * chunk, e = std::min(n, b + chunk);
    if (b >= e) break;
    th.emplace_back([&fn, b, e] { fn(b, e); });
  }
  for (auto &x : th) x.join();
}

struct HostField {
  uint32_t bit;
  int offset, size;
};
const HostField kHostFields[] = {
    {F_X, 0, 16},       {F_V, 16, 16},      {F_VPRED, 32, 16},  {F_A, 48, 16},
    {F_M, 64, 8},       {F_RHO, 72, 8},     {F_P, 80, 8},       {F_U, 88, 8},
    {F_UPRED, 96, 8},   {F_UDT, 104, 8},    {F_C, 112, 8},      {F_H, 120, 8},
    {F_WCOUNT, 128, 8}, {F_RHODH, 136, 8},  {F_ROTV, 144, 8},   {F_DIVV, 152, 8},
    {F_VSIG, 160, 8},   {F_HDT, 168, 8},    {F_DTNEXT, 176, 8}, {F_FROZEN, 184, 4},
    {F_MOVED, 188, 4},  {F_FLAGS, 208, 8},  {F_DBG, 216, 16},   {F_CELL, 200, 8},
};

uint32_t kernel_in(int k) {
  switch (k) {
  case SPH_DENSITY: return DEN_IN;
  case SPH_FORCE: return FOR_IN;
  case SPH_DRIFT: return DRIFT_IN;
  case SPH_KICK1: return KICK1_IN;
  default: return KICK2_IN;
  }
}
uint32_t kernel_out(int k) {
  switch (k) {
  case SPH_DENSITY: return DEN_OUT;
  case SPH_FORCE: return FOR_OUT;
  case SPH_DRIFT: return DRIFT_OUT;
  case SPH_KICK1: return KICK1_OUT;
  default: return KICK2_OUT;
  }
}

constexpr uint32_t kSoaFields = F_ALL_SOA & ~F_CELL; // fields with a SoA array

// grid.cpp:23-26
int grid_nx(int64_t n, int ppc) {
  double cell = std::sqrt(static_cast<double>(ppc) / static_cast<double>(std::max<int64_t>(n, 1)));
  return std::max(1, static_cast<int>(std::floor(1.0 / cell)));
}

// std::mt19937_64 (MT19937-64), grid.cpp:77 + unit_real grid.cpp:15-19.
struct Mt64 {
  uint64_t mt[312];
  int mti;
  explicit Mt64(uint64_t seed) {
    mt[0] = seed;
    for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
    mti = 312;
  }
  uint64_t next() {
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
    if (mti >= 312) {
      int i;
      for (i = 0; i < 156; ++i) {
        uint64_t x = (mt[i] & UM) | (mt[i + 1] & LM);
        mt[i] = mt[i + 156] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
      }
      for (; i < 311; ++i) {
        uint64_t x = (mt[i] & UM) | (mt[i + 1] & LM);
        mt[i] = mt[i - 156] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
      }
      uint64_t x = (mt[311] & UM) | (mt[0] & LM);
      mt[311] = mt[155] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
      mti = 0;
    }
    uint64_t x = mt[mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
  }
  double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

} // namespace

struct sph_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  // pipelined end-to-end step (sph_step_host): force chunks on two streams, per-chunk
  // kick2 + host-order compaction on `post`, device->host copies on `copy`
  cudaStream_t fs[2]{}, post = nullptr, copy = nullptr;
  cudaEvent_t pev[72]{};
  int pipeline = 1; // env SPH_B200_PIPELINE=0: serial force -> kick2 -> download
  static constexpr int kMaxPipeK = 32;
  int pipe_k = 16;  // env SPH_B200_PIPE_K: force chunks of the pipelined step (2..32); 16 vs 8: exposed tail 1.57 -> 1.04 ms
  int pipe_tail = 2; // env SPH_B200_PIPE_TAIL: shrinking last chunks (2: the last two half size)
  std::string err;
  int numerics = SPH_NUMERICS_FAST;
  int layout = SPH_LAYOUT_FROM_PATH;

  // geometry
  bool bound = false;
  int64_t n = 0;
  int nx = 0, ny = 0, ncells = 0;
  double cell_size = 0.0;
  bool identity_order = true; // slot s holds bound record s (no rebin since bind)

  // device state
  DevBuf<Particle> aos, aos_tmp;
  DevBuf<Particle> lin_recs; // sph_apply_records scratch (independent of the bound mirror)
  DevBuf<double2> f_x, f_v, f_vp, f_a, tmp2;
  DevBuf<double> f_m, f_rho, f_p, f_u, f_upred, f_udt, f_c, f_h, f_wc, f_rdh, f_rot, f_div,
      f_vsig, f_hdt, f_dtn, f_dbg0, tmp1;
  DevBuf<int32_t> f_frozen, f_moved;
  DevBuf<int64_t> f_flags, tmp8;
  // rebin by fix-up: the second SoA set the fused permute writes into (swapped in after)
  DevBuf<double2> g_x, g_v, g_vp, g_a;
  DevBuf<double> g_m, g_rho, g_p, g_u, g_upred, g_udt, g_c, g_h, g_wc, g_rdh, g_rot, g_div,
      g_vsig, g_hdt, g_dtn, g_dbg0;
  DevBuf<int32_t> g_frozen, g_moved;
  DevBuf<int64_t> g_flags;
  DevBuf<int> slot_cell, slot_cell_tmp, fx_moved, fx_mpos, fx_out, fx_in, fx_in_begin, fx_in_fill,
      fx_inlist, fx_new_begin, fx_perm;
  DevBuf<char> fx_scan;
  bool fixup_ok = false;   // slots in (cell, all_rank) order with slot_cell current (rebin_fixup)
  int rebin_fixup_on = 1;  // env SPH_B200_REBIN_FIXUP=0: every rebin sorts
  bool soa_alloc = false;
  SoaMirror soa{};

  DevBuf<int> cell_begin, cnt, pend_cnt, pend_cnt2, na_cell, ilist, pend_a, pend_b, host_idx, host_idx_tmp,
      cellnew, vals, vals_sorted, scalars;
  DevBuf<long long> all_rank, all_rank_tmp, pairs_dev, pairs_dev2; // {sum nl*na, particles}
  DevBuf<unsigned long long> fail_dev; // density: particles that hit the 30-round limit
  DevBuf<int> item_ctr;                 // density: persistent-round item counters
  // resident mirror: the AoS record fields without a SoA array (id, cell, dbg[1], spare) of
  // slot k live at aos[home[k]] while home_on (the fix-up rebin moves the map, not them)
  DevBuf<int> home, home_tmp;
  bool home_on = false;
  DevBuf<int> f2_ctr;                   // force2 persistent launches: item counters (per stream)
  DevBuf<unsigned long long> keys, keys_sorted;
  DevBuf<unsigned> cost_key, cost_key_sorted;
  DevBuf<unsigned char> owned;
  bool has_owned = false;
  DevBuf<int> cell_order, cell_order_in;
  DevBuf<Item> items0, items_a, items_b, items_c, items_d2, items_g;
  DevBuf<int> cnt_sp, cnt_dn;
  DevBuf<int> hdep;
  DevBuf<double> hcur, wc;
  DevBuf<unsigned char> rounds, again;
  DevBuf<float4> boxes;
  DevBuf<double2> jv_xy, jv_vv, jv_mg, jv_pv;
  DevBuf<double> jv_m, jv_c, jv2_fblk; // jv2_fblk: chunk-major force j-view
  DevBuf<double> jv2_x, jv2_y, jv2_m;   // density j-view
  DevBuf<double2> jv2_vv;
  size_t jv_blocks() const { return (size_t)n / 32 + (size_t)ncells + 2; }
  int force2 = 1; // FAST force on the resident SoA: issue-lean kernel (env SPH_B200_FORCE2=0: old)
  // lean density: lanes per particle in round 0 / rounds >= 1; rounds >= 1 use one lane per
  // particle in cells whose pending share exceeds den_dense_frac (r2, profiles/r2e_den_js1.txt:
  // 4 lanes / 0.5 against 2 / 0.35: C2 round 1 3.89 -> 3.45 ms, C4 within 0.4 %)
  int den_js0 = 1, den_js1 = 4;
  double den_dense_frac = 0.5;
  int den_dense_abs = 1024; // ... or whose pending count reaches this (env SPH_B200_DEN_DENSE_ABS;
                           // C3 round 1 15.1 -> 13.2 ms, C2 and C4 unchanged, r2g)
  bool dev_rounds = true; // density rounds >= 1 queued with device-side item counts (env SPH_B200_DEV_ROUNDS)
  // persistent pair sweeps (one warp per resident slot, items from an atomic counter in list
  // order): force -1.3 %, density round 0 -0.9 % against one CTA per item (r2d)
  bool persist0 = true;   // density round 0 (env SPH_B200_PERSIST0)
  bool f2_persist = true; // force2 (env SPH_B200_F2_PERSIST)
  bool cull = true; // FAST density: spatial j order + chunk culling (env SPH_B200_CULL=0 disables)
  DevBuf<char> dense, cub_tmp;
  PinnedBuf h_stage, h_small, h_items0;
  int n_items0 = 0;         // valid on the host after sync_items0()
  bool items0_pending = false; // the round-0 work list's count / pairs still in flight to the host
  bool force_pairs_pending = false;
  DevBuf<int> items0_n;        // its item count on the device (persistent sweeps read it there)
  DevBuf<long long> pairs0_dev; // {sum nl*na, listed particles} of the round-0 list
  bool need_rebin = false; // particles were appended: cell lists stale until sph_rebin
  DevBuf<unsigned char> dd_mask, dd_flag, sub_mask;
  DevBuf<int> sub_cnt;
  DevBuf<Item> items_sub;
  cudaStream_t own_stream = nullptr; // the stream sph_create made (sph_set_stream may replace `stream`)
  DevBuf<int> dd_sel, dd_cnt;
  DevBuf<int> mi_k, mi_off;
  DevBuf<char> mi_tmp;
  ItemsScratch mi{};
  const ItemsScratch *items_scratch() {
    mi_k.ensure(ncells);
    mi_off.ensure(ncells);
    const size_t tb = make_items_scratch_bytes(ncells);
    mi_tmp.ensure(tb);
    mi = ItemsScratch{mi_k.p, mi_off.p, mi_tmp.p, tb};
    launched(3); // counts + scan + write instead of one single-block kernel
    return &mi;
  }
  int64_t active_pairs = 0;
  int64_t listed0 = 0; // particles in the round-0 work list (owned cells' locals)

  // mirror state
  uint32_t dirty = 0;      // fields written on the device since the last host sync
  bool soa_valid = false;  // SoA arrays hold current values of every SoA field
  bool soa_ahead = false;  // SoA newer than AoS (resident mode)

  sph_stats stats{};
  int64_t launches = 0;
  cudaEvent_t ev[20]{};
  cudaEvent_t rev[8]{};    // density round kernels (first four rounds)
  double round_ms[4]{};

  ~sph_ctx() {
    for (auto &e : pev)
      if (e) cudaEventDestroy(e);
    for (auto &q : fs)
      if (q) cudaStreamDestroy(q);
    if (post) cudaStreamDestroy(post);
    if (copy) cudaStreamDestroy(copy);
    for (auto &e : ev)
      if (e) cudaEventDestroy(e);
    for (auto &e : rev)
      if (e) cudaEventDestroy(e);
    if (own_stream) cudaStreamDestroy(own_stream);
    aos.release(); aos_tmp.release(); lin_recs.release(); fail_dev.release();
    f_x.release(); f_v.release(); f_vp.release(); f_a.release(); tmp2.release();
    f_m.release(); f_rho.release(); f_p.release(); f_u.release(); f_upred.release();
    f_udt.release(); f_c.release(); f_h.release(); f_wc.release(); f_rdh.release();
    f_rot.release(); f_div.release(); f_vsig.release(); f_hdt.release(); f_dtn.release();
    f_dbg0.release(); tmp1.release(); f_frozen.release(); f_moved.release(); f_flags.release();
    tmp8.release(); cell_begin.release(); cnt.release(); pend_cnt.release(); pend_cnt2.release(); na_cell.release(); again.release();
    ilist.release(); pend_a.release(); pend_b.release(); host_idx.release();
    host_idx_tmp.release(); cellnew.release(); vals.release(); vals_sorted.release();
    scalars.release(); all_rank.release(); all_rank_tmp.release(); pairs_dev.release();
    keys.release(); keys_sorted.release(); cost_key.release(); cost_key_sorted.release();
    cell_order.release(); cell_order_in.release(); items0.release(); items_a.release();
    items_b.release(); hcur.release(); wc.release(); rounds.release(); dense.release();
    cub_tmp.release(); h_stage.release(); h_small.release(); owned.release();
    items0_n.release(); pairs0_dev.release(); h_items0.release();
    items_c.release(); items_d2.release(); cnt_sp.release(); cnt_dn.release(); pairs_dev2.release();
    item_ctr.release(); f2_ctr.release(); home.release(); home_tmp.release();
    items_g.release(); hdep.release(); sub_mask.release(); sub_cnt.release(); items_sub.release();
    dd_mask.release(); dd_flag.release(); dd_sel.release(); dd_cnt.release();
    mi_k.release(); mi_off.release(); mi_tmp.release();
    jv_xy.release(); jv_vv.release(); jv_mg.release(); jv_pv.release(); jv_m.release(); jv_c.release();
    jv2_fblk.release(); jv2_x.release(); jv2_y.release(); jv2_m.release(); jv2_vv.release();
    g_x.release(); g_v.release(); g_vp.release(); g_a.release(); g_m.release(); g_rho.release();
    g_p.release(); g_u.release(); g_upred.release(); g_udt.release(); g_c.release(); g_h.release();
    g_wc.release(); g_rdh.release(); g_rot.release(); g_div.release(); g_vsig.release();
    g_hdt.release(); g_dtn.release(); g_dbg0.release(); g_frozen.release(); g_moved.release();
    g_flags.release(); slot_cell.release(); slot_cell_tmp.release(); fx_moved.release();
    fx_mpos.release(); fx_out.release(); fx_in.release(); fx_in_begin.release();
    fx_in_fill.release(); fx_inlist.release(); fx_new_begin.release(); fx_perm.release();
    fx_scan.release();
  }

  Geom geom() const {
    Geom g;
    g.nx = nx;
    g.ny = ny;
    g.ncells = ncells;
    g.use_shift = (nx >= 5 && ny >= 5) ? 1 : 0;
    g.cell_size = cell_size;
    g.cell_begin = cell_begin.p;
    return g;
  }

  void ensure_soa() {
    const size_t N = (size_t)std::max<int64_t>(n, 1);
    f_x.ensure(N); f_v.ensure(N); f_vp.ensure(N); f_a.ensure(N);
    f_m.ensure(N); f_rho.ensure(N); f_p.ensure(N); f_u.ensure(N); f_upred.ensure(N);
    f_udt.ensure(N); f_c.ensure(N); f_h.ensure(N); f_wc.ensure(N); f_rdh.ensure(N);
    f_rot.ensure(N); f_div.ensure(N); f_vsig.ensure(N); f_hdt.ensure(N); f_dtn.ensure(N);
    f_dbg0.ensure(N); f_frozen.ensure(N); f_moved.ensure(N); f_flags.ensure(N);
    soa = SoaMirror{f_x.p, f_v.p, f_vp.p, f_a.p, f_m.p, f_rho.p, f_p.p, f_u.p, f_upred.p,
                    f_udt.p, f_c.p, f_h.p, f_wc.p, f_rdh.p, f_rot.p, f_div.p, f_vsig.p,
                    f_hdt.p, f_dtn.p, f_dbg0.p, f_frozen.p, f_moved.p, f_flags.p};
    soa_alloc = true;
  }

  SoaMirror soa_at(int64_t off) const {
    SoaMirror f = soa;
    f.x += off; f.v += off; f.vp += off; f.a += off; f.m += off; f.rho += off; f.p += off;
    f.u += off; f.u_pred += off; f.u_dt += off; f.c += off; f.h += off; f.wcount += off;
    f.rho_dh += off; f.rot_v += off; f.div_v += off; f.v_sig += off; f.h_dt += off;
    f.dt_next += off; f.dbg0 += off; f.frozen += off; f.moved += off; f.flags += off;
    return f;
  }

  // Room for nn particles in every per-slot array that holds state (the first n kept).
  void grow_state(int64_t nn) {
    const size_t N = (size_t)nn, K = (size_t)n;
    aos.reserve_keep(N, K, stream);
    all_rank.reserve_keep(N, K, stream);
    host_idx.reserve_keep(N, K, stream);
    if (soa_alloc) {
      f_x.reserve_keep(N, K, stream); f_v.reserve_keep(N, K, stream); f_vp.reserve_keep(N, K, stream);
      f_a.reserve_keep(N, K, stream); f_m.reserve_keep(N, K, stream); f_rho.reserve_keep(N, K, stream);
      f_p.reserve_keep(N, K, stream); f_u.reserve_keep(N, K, stream); f_upred.reserve_keep(N, K, stream);
      f_udt.reserve_keep(N, K, stream); f_c.reserve_keep(N, K, stream); f_h.reserve_keep(N, K, stream);
      f_wc.reserve_keep(N, K, stream); f_rdh.reserve_keep(N, K, stream); f_rot.reserve_keep(N, K, stream);
      f_div.reserve_keep(N, K, stream); f_vsig.reserve_keep(N, K, stream); f_hdt.reserve_keep(N, K, stream);
      f_dtn.reserve_keep(N, K, stream); f_dbg0.reserve_keep(N, K, stream);
      f_frozen.reserve_keep(N, K, stream); f_moved.reserve_keep(N, K, stream);
      f_flags.reserve_keep(N, K, stream);
      soa = SoaMirror{f_x.p, f_v.p, f_vp.p, f_a.p, f_m.p, f_rho.p, f_p.p, f_u.p, f_upred.p,
                      f_udt.p, f_c.p, f_h.p, f_wc.p, f_rdh.p, f_rot.p, f_div.p, f_vsig.p,
                      f_hdt.p, f_dtn.p, f_dbg0.p, f_frozen.p, f_moved.p, f_flags.p};
    }
  }

  void alloc_for(int64_t nn, int nc) {
    const size_t N = (size_t)std::max<int64_t>(nn, 1);
    aos.ensure(N);
    cell_begin.ensure(nc + 1);
    cnt.ensure(nc);
    pend_cnt.ensure(nc);
    pend_cnt2.ensure(nc);
    again.ensure(N);
    na_cell.ensure(nc);
    ilist.ensure(N);
    pend_a.ensure(N);
    pend_b.ensure(N);
    host_idx.ensure(N);
    all_rank.ensure(N);
    hcur.ensure(N);
    rounds.ensure(N);
    scalars.ensure(4);
    pairs_dev.ensure(2);
    // worst case items: one per cell + n / kTI
    const size_t it = (size_t)nc + N / kTI + 1;
    items0.ensure(it);
    items_a.ensure(it);
    items_b.ensure(it);
    h_small.ensure(64);
  }

  void launched(int k = 1) { launches += k; }

  // Work list + derived per-cell data after the slot order changed.
  void rebuild_worklist() {
    // per-cell counts, then the cell processing order: descending cost bucket, stable, so
    // heavy cells (variable ppc) are scheduled first (LPT) while cells of similar cost keep
    // their grid order (L2 reuse of shared neighbour cells)
    cost_key.ensure(ncells);
    cost_key_sorted.ensure(ncells);
    cell_order_in.ensure(ncells);
    cell_order.ensure(ncells);
    launch_cell_counts(na_cell.p, cnt.p, cost_key.p, cell_order_in.p, cell_begin.p, nx, ny, stream);
    if (has_owned) {
      launch_mask_counts(cnt.p, cost_key.p, owned.p, ncells, stream); // halo cells: no items
      launched();
    }
    {
      size_t tb = 0;
      CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, cost_key.p, cost_key_sorted.p,
                                                   cell_order_in.p, cell_order.p, ncells, 0, 10,
                                                   stream));
      cub_tmp.ensure(tb);
      CK(cub::DeviceRadixSort::SortPairsDescending(cub_tmp.p, tb, cost_key.p, cost_key_sorted.p,
                                                   cell_order_in.p, cell_order.p, ncells, 0, 10,
                                                   stream));
      launched(2);
    }
    const bool aos_src = !soa_ahead;
    launch_spatial_order(ilist.p, aos.p, soa, aos_src, cell_begin.p, ncells, nx, ny, stream);
    items0_n.ensure(1);
    pairs0_dev.ensure(2);
    h_items0.ensure(32);
    launch_make_items(items0.p, items0_n.p, pairs0_dev.p, cnt.p, cell_begin.p, na_cell.p,
                      cell_order.p, ncells, stream, kTI, items_scratch());
    launched(3);
    // the count travels to the host behind the step's work: the persistent density round 0
    // and force sweep read it on the device, everything else calls sync_items0() first
    CK(cudaMemcpyAsync(h_items0.p, items0_n.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync((char *)h_items0.p + 8, pairs0_dev.p, 2 * sizeof(long long),
                       cudaMemcpyDeviceToHost, stream));
    items0_pending = true;
  }

  // The round-0 work list's count and pair totals on the host (synchronises the stream if
  // they are still in flight).
  void sync_items0() {
    if (!items0_pending) return;
    CK(cudaStreamSynchronize(stream));
    n_items0 = *(const int *)h_items0.p;
    active_pairs = *(const long long *)((const char *)h_items0.p + 8);
    listed0 = *(const long long *)((const char *)h_items0.p + 16);
    stats.active_pairs = active_pairs;
    if (force_pairs_pending) stats.force_pairs = active_pairs;
    items0_pending = force_pairs_pending = false;
  }

  // ---- mirror coherence ----
  // the record tails back into slot order (aos[k] holds slot k's id, cell, dbg[1], spare)
  void normalize_tails() {
    if (!home_on) return;
    aos_tmp.ensure(n);
    launch_permute_record_tails(aos_tmp.p, aos.p, home.p, (int)n, stream);
    launched();
    std::swap(aos.p, aos_tmp.p);
    std::swap(aos.cap, aos_tmp.cap);
    home_on = false;
  }
  void make_aos_current() {
    normalize_tails();
    if (soa_ahead) {
      launch_scatter(aos.p, soa, (int)n, kSoaFields, stream);
      launched();
      soa_ahead = false;
    }
  }
  void make_soa_current() {
    ensure_soa();
    if (!soa_valid) {
      normalize_tails();
      launch_gather(aos.p, soa, (int)n, kSoaFields, stream);
      launched();
      soa_valid = true;
    }
  }

  // ---- sweeps ----
  int mode_for(int path) const {
    if (layout == SPH_LAYOUT_FROM_PATH) return path == SPH_PATH_SOA_VIEW ? SPH_LAYOUT_CONVERT : SPH_LAYOUT_AOS;
    return layout;
  }

  void run_density(bool use_aos, bool exact, const Params &par, bool meanw) {
    DenArgs A{};
    A.g = geom();
    A.target = par.target_wcount;
    A.h_max = cell_size / kSupport; // kernels.cpp:542
    A.aos = aos.p;
    A.soa = soa;
    A.hcur = hcur.p;
    A.again = again.p;
    A.rounds_out = rounds.p;
    A.wc_out = wc.p;
    if (!exact && !meanw && cull) {
      boxes.ensure((size_t)n / 32 + (size_t)ncells + 2);
      launch_chunk_boxes(boxes.p, ilist.p, aos.p, soa, use_aos, cell_begin.p, ncells, stream);
      launched();
      A.boxes = boxes.p;
      A.jlist = ilist.p;
      if (force2 && A.g.use_shift) { // issue-lean density (any layout)
        jv2_x.ensure(n); jv2_y.ensure(n); jv2_m.ensure(n); jv2_vv.ensure(n);
        A.jv2 = D2View{jv2_x.p, jv2_y.p, jv2_m.p, jv2_vv.p};
        // the AoS arm stages its j's from the records (no j-view)
        if (!use_aos) launch_jview_density2(A.jv2, ilist.p, aos.p, soa, use_aos, (int)n, stream);
      } else {
        jv_xy.ensure(n); jv_vv.ensure(n); jv_m.ensure(n);
        launch_jview_density(jv_xy.p, jv_vv.p, jv_m.p, ilist.p, aos.p, soa, use_aos, (int)n, stream);
        A.jv.xy = jv_xy.p;
        A.jv.vv = jv_vv.p;
        A.jv.m = jv_m.p;
      }
      launched();
    }
    const bool lean = A.jv2.x != nullptr;
    // device-counted rounds (see below) and a persistent round 0 that reads its item count on
    // the device: no host synchronisation between the rebin and the end of round 2
    const bool spec = lean && den_js1 > 1 && !exact && !meanw && dev_rounds;
    const bool dev0 = spec && persist0 && den_js0 <= 1;
    if (!dev0) sync_items0();
    const int js0 = lean ? std::max(1, std::min(4, den_js0)) : 1;
    const int js1 = lean ? std::max(1, std::min(8, den_js1)) : 1;
    const Item *items = items0.p;
    const int *list = ilist.p;
    const int *cnt_cur = cnt.p; // entries of `list` per cell (round 0: every local)
    int nitems = n_items0;
    items_a.ensure((size_t)ncells + (size_t)n / (kTI / std::max(js0, js1)) + 1);
    items_b.ensure((size_t)ncells + (size_t)n / (kTI / std::max(js0, js1)) + 1);
    if (js0 > 1) { // round-0 items of 32/js0 particles
      launch_make_items(items_b.p, scalars.p, pairs_dev.p, cnt.p, cell_begin.p, na_cell.p,
                        cell_order.p, ncells, stream, kTI / js0, items_scratch());
      launched();
      CK(cudaMemcpyAsync(h_small.p, scalars.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
      CK(cudaStreamSynchronize(stream));
      nitems = *(int *)h_small.p;
      items = items_b.p;
    }
    int64_t pairs = active_pairs, pairs_total = 0;
    int64_t pending = listed0, updates = 0;
    int max_round = 0;
    if (!meanw) {
      fail_dev.ensure(1);
      CK(cudaMemsetAsync(fail_dev.p, 0, sizeof(unsigned long long), stream));
      A.fail_count = fail_dev.p;
    }
    for (double &v : round_ms) v = 0.0;
    int *pend_out = pend_a.p;
    int *cnt_out = pend_cnt.p;
    Item *items_next = items_a.p;
    // rounds >= 1 (lean kernel, js1 > 1): j-slices pay while a cell's pending particles are
    // sparse (their warps' boxes stay small); when most of a cell is pending, full warps are
    // compact already and one lane per particle is faster (2^24: round 1 93.3 -> 91.0 ms; at
    // 2^21, ~12 % pending, two lanes win: 4.9 -> 4.2 ms). The choice is made per cell from
    // the cell's own pending share, so a cell's summation order (and its FAST result) does
    // not depend on which other cells a context holds (k decomposed ranks == one rank).
    const bool split = lean && js1 > 1;
    const Item *items_d = nullptr; // the round's one-lane-per-particle items (dense cells)
    int nitems_d = 0;
    Item *items_next_d = items_c.p;
    if (split) {
      items_c.ensure((size_t)ncells + (size_t)n / kTI + 1);
      items_d2.ensure((size_t)ncells + (size_t)n / kTI + 1);
      items_next_d = items_c.p;
      cnt_sp.ensure(ncells);
      cnt_dn.ensure(ncells);
      pairs_dev2.ensure(2);
    }
    // Device-counted rounds (lean FAST density with the dense/sparse split): rounds
    // 1 .. kSpecRounds-1 are queued right behind round 0 without the host learning their
    // item counts; their kernels are persistent and read the count that the previous
    // round's make_items left in device memory (an empty round costs one short launch).
    // The host synchronises once after round kSpecRounds-1 and continues round by round
    // only if particles are still pending (rare: two rounds are typical at dt = 1e-4).
    constexpr int kSpecRounds = 3;
    item_ctr.ensure(2);
    if (spec) {
      h_small.ensure(64 + 64 * kSpecRounds);
    }
    auto slot = [&](int r) { return (char *)h_small.p + 64 + 64 * r; };
    bool host_known = !dev0; // nitems, nitems_d, pairs, pending describe round r
    for (int r = 0; r < 30; ++r) {
      if (host_known && nitems <= 0 && nitems_d <= 0) break;
      const bool devc = spec && r > 0 && r < kSpecRounds;
      A.items = items;
      A.list = list;
      A.round = r;
      A.jslices = r == 0 ? js0 : js1;
      A.n_items_dev = devc ? scalars.p : (r == 0 && dev0) ? items0_n.p : nullptr;
      A.item_ctr = devc || (r == 0 && persist0 && lean && !exact && !meanw) ? item_ctr.p : nullptr;
      if (meanw) {
        launch_density_exact(A, nitems, use_aos, true, stream);
        launched();
        break;
      }
      if (r < 4) CK(cudaEventRecord(rev[2 * r], stream));
      if (exact) launch_density_exact(A, nitems, use_aos, false, stream);
      else launch_density_fast(A, nitems, use_aos, stream);
      launched();
      if (devc || nitems_d > 0) { // same round, dense cells, one lane per particle
        DenArgs D = A;
        D.items = items_d;
        D.jslices = 1;
        D.n_items_dev = devc ? scalars.p + 1 : nullptr;
        D.item_ctr = devc ? item_ctr.p + 1 : nullptr;
        launch_density_fast(D, nitems_d, use_aos, stream);
        launched();
      }
      if (r < 4) CK(cudaEventRecord(rev[2 * r + 1], stream));
      launch_compact_pending(pend_out, cnt_out, list, cnt_cur, again.p, cell_begin.p, ncells,
                             stream);
      if (host_known) {
        pairs_total += pairs;
        updates += pending;
        max_round = r + 1;
      }
      if (split) {
        launch_split_pending(cnt_sp.p, cnt_dn.p, cnt_out, cnt.p, den_dense_frac, den_dense_abs, ncells,
                             stream);
        launch_make_items(items_next, scalars.p, pairs_dev.p, cnt_sp.p, cell_begin.p, na_cell.p,
                          cell_order.p, ncells, stream, kTI / js1, items_scratch());
        launch_make_items(items_next_d, scalars.p + 1, pairs_dev2.p, cnt_dn.p, cell_begin.p,
                          na_cell.p, cell_order.p, ncells, stream, kTI, items_scratch());
        launched(8);
        char *hs = spec && r < kSpecRounds ? slot(r) : (char *)h_small.p;
        CK(cudaMemcpyAsync(hs, scalars.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, stream));
        CK(cudaMemcpyAsync(hs + 8, pairs_dev.p, 2 * sizeof(long long), cudaMemcpyDeviceToHost,
                           stream));
        CK(cudaMemcpyAsync(hs + 24, pairs_dev2.p, 2 * sizeof(long long), cudaMemcpyDeviceToHost,
                           stream));
        const bool queue_next = spec && r + 1 < kSpecRounds;
        if (!queue_next) {
          CK(cudaStreamSynchronize(stream));
          if (spec && r + 1 == kSpecRounds) {
            // account the device-counted rounds 0 .. r now that their counts are on the host
            if (dev0) {
              sync_items0(); // (the stream is idle: no wait)
              if (n_items0 > 0) {
                pairs_total += active_pairs;
                updates += listed0;
                max_round = 1;
              }
            }
            for (int k = 1; k <= r; ++k) {
              const char *q = slot(k - 1);
              if (((const int *)q)[0] <= 0 && ((const int *)q)[1] <= 0) break;
              pairs_total += *(const long long *)(q + 8) + *(const long long *)(q + 24);
              updates += *(const long long *)(q + 16) + *(const long long *)(q + 32);
              max_round = k + 1;
            }
          }
        }
        host_known = !queue_next;
        if (host_known) {
          nitems = ((int *)hs)[0];
          nitems_d = ((int *)hs)[1];
          pairs = *(long long *)(hs + 8) + *(long long *)(hs + 24);
          pending = *(long long *)(hs + 16) + *(long long *)(hs + 32);
        }
      } else {
        launch_make_items(items_next, scalars.p, pairs_dev.p, cnt_out, cell_begin.p, na_cell.p,
                          cell_order.p, ncells, stream, kTI / js1, items_scratch());
        launched(3);
        CK(cudaMemcpyAsync(h_small.p, scalars.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
        CK(cudaMemcpyAsync((char *)h_small.p + 8, pairs_dev.p, 2 * sizeof(long long),
                           cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        nitems = *(int *)h_small.p;
        pairs = *(long long *)((char *)h_small.p + 8);
        pending = *(long long *)((char *)h_small.p + 16);
      }
      if (host_known) // the rounds since the last synchronisation have completed
        for (int k = 0; k <= r && k < 4; ++k)
          if (round_ms[k] == 0.0 && k < max_round) {
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, rev[2 * k], rev[2 * k + 1]));
            round_ms[k] = ms;
          }
      // next round reads what this one produced
      items = items_next;
      items_d = items_next_d;
      list = pend_out;
      cnt_cur = cnt_out;
      items_next = (items_next == items_a.p) ? items_b.p : items_a.p;
      items_next_d = (items_next_d == items_c.p) ? items_d2.p : items_c.p;
      pend_out = (pend_out == pend_a.p) ? pend_b.p : pend_a.p;
      cnt_out = (cnt_out == pend_cnt.p) ? pend_cnt2.p : pend_cnt.p;
    }
    if (!meanw) {
      unsigned long long fails = 0;
      CK(cudaMemcpyAsync(&fails, fail_dev.p, sizeof fails, cudaMemcpyDeviceToHost, stream));
      CK(cudaStreamSynchronize(stream));
      stats.density_pairs = pairs_total;
      stats.density_updates = updates;
      stats.density_failures = (int64_t)fails;
      stats.density_rounds = max_round;
      for (int k = 0; k < 4; ++k) stats.density_round_ms[k] = round_ms[k];
    }
  }

  void run_force(bool use_aos, bool exact, const Params &par, const Item *items = nullptr,
                 int nitems = -1) {
    const bool dev_count = !items && items0_pending && f2_persist && !exact && cull && force2 &&
                           geom().use_shift;
    if (!items) {
      if (!dev_count) sync_items0();
      items = items0.p;
      nitems = n_items0;
    }
    ForArgs A{};
    A.g = geom();
    A.items = items;
    A.list = ilist.p;
    A.grav = par.grav;
    A.aos = aos.p;
    A.soa = soa;
    if (!exact && cull && force2 && A.g.use_shift) {
      // issue-lean kernel (spatial j order, far chunks gravity-only), any layout
      boxes.ensure((size_t)n / 32 + (size_t)ncells + 2);
      launch_chunk_boxes(boxes.p, ilist.p, aos.p, soa, use_aos, cell_begin.p, ncells, stream);
      jv2_fblk.ensure(jv_blocks() * kF2Blk);
      F2Args B{};
      B.g = A.g;
      B.items = items;
      B.list = ilist.p;
      B.grav = par.grav;
      B.aos = use_aos ? aos.p : nullptr;
      B.soa = soa;
      B.boxes = boxes.p;
      B.jv = F2View{jv2_fblk.p};
      if (f2_persist) {
        f2_ctr.ensure(2);
        B.item_ctr = f2_ctr.p;
      }
      if (dev_count) B.n_items_dev = items0_n.p; // persistent: the count is read on the device
      launch_force2(B, nitems, (int)n, stream);
      launched(3);
      if (dev_count) force_pairs_pending = true;
      else stats.force_pairs = active_pairs;
      return;
    }
    if (!exact && cull) { // spatial j order + far-chunk gravity-only path
      boxes.ensure((size_t)n / 32 + (size_t)ncells + 2);
      launch_chunk_boxes(boxes.p, ilist.p, aos.p, soa, use_aos, cell_begin.p, ncells, stream);
      jv_xy.ensure(n); jv_vv.ensure(n); jv_mg.ensure(n); jv_pv.ensure(n); jv_c.ensure(n);
      launch_jview_force(jv_xy.p, jv_vv.p, jv_mg.p, jv_pv.p, jv_c.p, ilist.p, aos.p, soa, use_aos,
                         (int)n, par.grav, stream);
      launched(2);
      A.boxes = boxes.p;
      A.jlist = ilist.p;
      A.jv.xy = jv_xy.p;
      A.jv.vv = jv_vv.p;
      A.jv.mg = jv_mg.p;
      A.jv.pv = jv_pv.p;
      A.jv.c = jv_c.p;
    }
    if (exact) launch_force_exact(A, nitems, use_aos, stream);
    else launch_force_fast(A, nitems, use_aos, stream);
    launched();
    stats.force_pairs = active_pairs;
  }

  bool can_pipeline(bool contig) const {
    return pipeline && numerics == SPH_NUMERICS_FAST && cull && force2 && !has_owned &&
           mode_for(SPH_PATH_AOS_BASELINE) == SPH_LAYOUT_RESIDENT && nx >= 5 && ny >= 5 &&
           n >= 4096 && contig;
  }

  // force -> kick2 -> download for host records at `host` (contiguous, bound order), with
  // the device->host copy of finished particles overlapping the rest of the force sweep.
  // The force sweep runs as K chunks of whole cells in grid (slot) order; chunk f finishes
  // slots [sb[f], sb[f+1]). After each chunk, kick2 and the host-order compaction of its
  // slots run on `post`; host chunk g (a contiguous range of records) is copied as soon as
  // the last force chunk holding one of its particles is through `post`. Times (ms):
  // out[0] force (first chunk start -> last chunk end), out[1] the exposed tail.
  void force_kick2_download_pipelined(void *host, const Params &par, float out[2]) {
    constexpr int G = 64;
    if (!fs[0]) {
      for (auto &q : fs) CK(cudaStreamCreateWithFlags(&q, cudaStreamNonBlocking));
      // kick2/compaction CTAs must not queue behind the force chunks' CTAs
      int lo = 0, hi = 0;
      CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      CK(cudaStreamCreateWithPriority(&post, cudaStreamNonBlocking, hi));
      CK(cudaStreamCreateWithPriority(&copy, cudaStreamNonBlocking, hi));
      for (auto &e : pev) CK(cudaEventCreate(&e));
    }
    make_soa_current();
    // grid-order items and the per-cell item prefix (host)
    items_g.ensure((size_t)ncells + (size_t)n / kTI + 1);
    launch_make_items(items_g.p, scalars.p, pairs_dev.p, cnt.p, cell_begin.p, na_cell.p, nullptr,
                      ncells, stream, kTI, items_scratch());
    launched();
    std::vector<int> cb(ncells + 1);
    CK(cudaMemcpyAsync(cb.data(), cell_begin.p, sizeof(int) * (ncells + 1), cudaMemcpyDeviceToHost,
                       stream));
    CK(cudaStreamSynchronize(stream));
    std::vector<int> kpre(ncells + 1, 0); // items in cells < c
    int maxc = 0;
    for (int c = 0; c < ncells; ++c) {
      kpre[c + 1] = kpre[c] + (cb[c + 1] - cb[c] + kTI - 1) / kTI;
      maxc = std::max(maxc, cb[c + 1] - cb[c]);
    }
    // chunk count: pipe_k on a near-uniform box; on a variable-ppc box (densest cell > 2x the
    // mean) at most 8, since chunks of very unequal work leave one of the two force streams
    // idle (measured, config 3: 16 chunks 150.3 ms vs 8 chunks 146.3 ms end to end)
    const int K = (double)maxc > 2.0 * n / std::max(1, ncells) ? std::min(pipe_k, 8) : pipe_k;
    // K chunks of whole cells with ~equal particle counts (equal-work chunks measured worse:
    // the last chunk's records, whose copy is the exposed tail, grow)
    ChunkBounds B{};
    B.k = K;
    int kb[kMaxPipeK + 1];
    {
      // the last T chunks shrink (1/2, 1/4, ... of a full one, the last two equal): the last
      // chunk's records are the exposed copy (T = 2: the last two half size)
      const int T = std::max(1, std::min(pipe_tail, K - 1));
      double w[kMaxPipeK];
      double tot = 0.0;
      for (int f = 0; f < K; ++f) {
        const int t = f - (K - T); // 0 .. T-1 in the tail
        w[f] = (t < 0 || T == 1) ? 1.0 : std::ldexp(1.0, -(std::min(t, T - 2) + 1));
        tot += w[f];
      }
      int c = 0;
      double acc = 0.0;
      for (int f = 0; f <= K; ++f) {
        const long long target = (long long)std::llround((double)n * acc / tot);
        while (c < ncells && cb[c] < target) ++c;
        if (f == K) c = ncells;
        B.s[f] = cb[c];
        kb[f] = kpre[c];
        if (f < K) acc += w[f];
      }
    }
    // host chunk -> last force chunk
    const int hsz = (int)((n + G - 1) / G);
    hdep.ensure(G);
    CK(cudaMemsetAsync(hdep.p, 0, sizeof(int) * G, stream));
    launch_host_chunk_dep(hdep.p, host_idx.p, (int)n, hsz, B, stream);
    launched();
    int dep[G];
    CK(cudaMemcpyAsync(dep, hdep.p, sizeof dep, cudaMemcpyDeviceToHost, stream));
    // force prologue: chunk boxes + j-view (main stream)
    boxes.ensure((size_t)n / 32 + (size_t)ncells + 2);
    launch_chunk_boxes(boxes.p, ilist.p, aos.p, soa, false, cell_begin.p, ncells, stream);
    jv2_fblk.ensure(jv_blocks() * kF2Blk);
    F2Args A{};
    A.g = geom();
    A.list = ilist.p;
    A.grav = par.grav;
    A.soa = soa;
    A.boxes = boxes.p;
    A.jv = F2View{jv2_fblk.p};
    A.items = items_g.p;
    launch_force2(A, 0, (int)n, stream); // j-view only
    launched(2);
    CK(cudaStreamSynchronize(stream)); // dep[] on the host
    cudaEvent_t e_pre = pev[0];
    CK(cudaEventRecord(e_pre, stream));
    dense.ensure((size_t)n * SPH_RECORD_SIZE);
    Particle *dn = reinterpret_cast<Particle *>(dense.p);
    for (int f = 0; f < K; ++f) {
      cudaStream_t q = fs[f & 1];
      if (f < 2) CK(cudaStreamWaitEvent(q, e_pre, 0));
      A.items = items_g.p + kb[f];
      if (f2_persist) { // one counter per force stream
        f2_ctr.ensure(2);
        A.item_ctr = f2_ctr.p + (f & 1);
      }
      launch_force2(A, kb[f + 1] - kb[f], 0, q);
      launched();
      CK(cudaEventRecord(pev[1 + f], q)); // force chunk f done
      CK(cudaStreamWaitEvent(post, pev[1 + f], 0));
      const int s0 = B.s[f], s1 = B.s[f + 1];
      if (s1 > s0) {
        SoaMirror o = soa_at(s0);
        launch_linear(SPH_KICK2, false, aos.p + s0, o, s1 - s0, par, post);
        launch_compact_soa(dn, aos.p, soa, host_idx.p, home_on ? home.p : nullptr, s0, s1, post);
        launched(2);
      }
      CK(cudaEventRecord(pev[1 + K + f], post)); // slots of chunk f final in `dense`
    }
    // copies in order of readiness
    int order[G];
    for (int g = 0; g < G; ++g) order[g] = g;
    std::stable_sort(order, order + G, [&](int a, int b) { return dep[a] < dep[b]; });
    int waited = -1;
    for (int t = 0; t < G; ++t) {
      const int g = order[t];
      const int64_t h0 = (int64_t)g * hsz, h1 = std::min<int64_t>(n, h0 + hsz);
      if (h1 <= h0) continue;
      if (dep[g] > waited) {
        CK(cudaStreamWaitEvent(copy, pev[1 + K + dep[g]], 0));
        waited = dep[g];
      }
      CK(cudaMemcpyAsync(static_cast<char *>(host) + h0 * SPH_RECORD_SIZE,
                         reinterpret_cast<char *>(dn + h0), (size_t)(h1 - h0) * SPH_RECORD_SIZE,
                         cudaMemcpyDeviceToHost, copy));
    }
    // join: the main stream waits for the last force chunks, post and copy
    CK(cudaEventRecord(pev[2 * K + 1], copy));
    CK(cudaEventRecord(pev[2 * K + 2], post));
    CK(cudaStreamWaitEvent(stream, pev[K - 1], 0));
    CK(cudaStreamWaitEvent(stream, pev[K], 0));
    CK(cudaStreamWaitEvent(stream, pev[2 * K + 1], 0));
    CK(cudaStreamWaitEvent(stream, pev[2 * K + 2], 0));
    CK(cudaEventRecord(pev[2 * K + 3], stream));
    CK(cudaEventSynchronize(pev[2 * K + 3]));
    float a0 = 0, a1 = 0, t = 0;
    CK(cudaEventElapsedTime(&a0, e_pre, pev[K - 1])); // the last chunk of each force stream
    CK(cudaEventElapsedTime(&a1, e_pre, pev[K]));
    CK(cudaEventElapsedTime(&t, e_pre, pev[2 * K + 3]));
    out[0] = std::max(a0, a1);
    out[1] = t - out[0]; // exposed kick2 / copy tail
    stats.force_pairs = active_pairs;
    soa_ahead = true;
    soa_valid = true;
    dirty = 0;
  }

  SoaMirror soa_at(int s0) const {
    SoaMirror o = soa;
    o.x += s0; o.v += s0; o.vp += s0; o.a += s0; o.m += s0; o.rho += s0; o.p += s0; o.u += s0;
    o.u_pred += s0; o.u_dt += s0; o.c += s0; o.h += s0; o.wcount += s0; o.rho_dh += s0;
    o.rot_v += s0; o.div_v += s0; o.v_sig += s0; o.h_dt += s0; o.dt_next += s0; o.dbg0 += s0;
    o.frozen += s0; o.moved += s0; o.flags += s0;
    return o;
  }

  // ---- domain decomposition (device-resident slabs, decomp.py) ----
  // Slots whose column clamp(floor(x * nx)) is set in `col_mask` (or clear, `invert`), in
  // slot order, into dd_sel; returns the count.
  int64_t dd_select(const uint8_t *col_mask, bool invert) {
    dd_mask.ensure(nx);
    CK(cudaMemcpyAsync(dd_mask.p, col_mask, nx, cudaMemcpyHostToDevice, stream));
    dd_flag.ensure(n);
    dd_sel.ensure(n);
    dd_cnt.ensure(1);
    const bool aos_src = !(soa_ahead || soa_valid);
    launch_col_flags(dd_flag.p, aos.p, soa, aos_src, dd_mask.p, (int)n, nx, invert ? 1 : 0, stream);
    size_t tb = 0;
    thrust::counting_iterator<int> it(0);
    CK(cub::DeviceSelect::Flagged(nullptr, tb, it, dd_flag.p, dd_sel.p, dd_cnt.p, (int)n, stream));
    cub_tmp.ensure(tb);
    CK(cub::DeviceSelect::Flagged(cub_tmp.p, tb, it, dd_flag.p, dd_sel.p, dd_cnt.p, (int)n, stream));
    launched(2);
    int cnt_h = 0;
    CK(cudaMemcpyAsync(&cnt_h, dd_cnt.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    return cnt_h;
  }
  int64_t dd_export(const uint8_t *col_mask, Particle *out, long long *ranks_out, int64_t cap) {
    if (n == 0) return 0;
    normalize_tails();
    const int64_t m = dd_select(col_mask, false);
    if (m > cap) throw ArgError{"export buffer too small"};
    if (soa_ahead) // resident: assemble the selected records from the SoA mirror + tails
      launch_export_soa(out, aos.p, soa, dd_sel.p, (int)m, stream);
    else
      launch_permute<Particle>(out, aos.p, dd_sel.p, (int)m, stream);
    if (ranks_out) launch_permute<long long>(ranks_out, all_rank.p, dd_sel.p, (int)m, stream);
    launched(2);
    CK(cudaStreamSynchronize(stream));
    return m;
  }
  void dd_reset_host_order() {
    host_idx.ensure(n);
    launch_iota(host_idx.p, (int)n, stream);
    launched();
    identity_order = true;
  }
  void dd_remove(const uint8_t *col_mask) {
    if (n == 0) return;
    normalize_tails();
    const int64_t keep = dd_select(col_mask, true);
    if (keep == n) return;
    apply_perm(dd_sel.p, keep); // (sel is read before the buffers it indexes are swapped)
    n = keep;
    fixup_ok = false;
    dd_reset_host_order();
    need_rebin = true;
    CK(cudaStreamSynchronize(stream));
  }
  void dd_append(const Particle *recs, const long long *ranks, int64_t m) {
    if (m <= 0) return;
    normalize_tails();
    if (n + m >= (1LL << 31)) throw ArgError{"particle count out of range"};
    if (soa_ahead || soa_valid) {
      // resident: the records go to the AoS mirror and their fields straight into the SoA
      // mirror at slots [n, n + m); the mirror state (SoA ahead or both valid) is kept
      ensure_soa();
      grow_state(n + m);
      CK(cudaMemcpyAsync(aos.p + n, recs, sizeof(Particle) * m, cudaMemcpyDeviceToDevice, stream));
      CK(cudaMemcpyAsync(all_rank.p + n, ranks, sizeof(long long) * m, cudaMemcpyDeviceToDevice, stream));
      launch_gather(aos.p + n, soa_at(n), (int)m, kSoaFields, stream);
      launched();
      n += m;
      fixup_ok = false;
      alloc_for(n, ncells);
      dd_reset_host_order();
      need_rebin = true;
      CK(cudaStreamSynchronize(stream));
      return;
    }
    make_aos_current();
    const int64_t nn = n + m;
    aos_tmp.ensure(nn);
    if (n) CK(cudaMemcpyAsync(aos_tmp.p, aos.p, sizeof(Particle) * n, cudaMemcpyDeviceToDevice, stream));
    CK(cudaMemcpyAsync(aos_tmp.p + n, recs, sizeof(Particle) * m, cudaMemcpyDeviceToDevice, stream));
    std::swap(aos.p, aos_tmp.p);
    std::swap(aos.cap, aos_tmp.cap);
    all_rank_tmp.ensure(nn);
    if (n) CK(cudaMemcpyAsync(all_rank_tmp.p, all_rank.p, sizeof(long long) * n, cudaMemcpyDeviceToDevice, stream));
    CK(cudaMemcpyAsync(all_rank_tmp.p + n, ranks, sizeof(long long) * m, cudaMemcpyDeviceToDevice, stream));
    std::swap(all_rank.p, all_rank_tmp.p);
    std::swap(all_rank.cap, all_rank_tmp.cap);
    CK(cudaStreamSynchronize(stream));
    n = nn;
    fixup_ok = false;
    alloc_for(n, ncells); // scratch sized for the new count (aos / all_rank already are)
    soa_valid = false;    // the SoA is re-gathered from the AoS by the next resident sweep
    soa_ahead = false;
    dd_reset_host_order();
    need_rebin = true;
    CK(cudaStreamSynchronize(stream));
  }
  int64_t dd_export_rho(const uint8_t *col_mask, double *out, int64_t cap) {
    if (n == 0) return 0;
    const int64_t m = dd_select(col_mask, false);
    if (m > cap) throw ArgError{"export buffer too small"};
    if (soa_ahead || soa_valid) {
      launch_permute<double>(out, soa.rho, dd_sel.p, (int)m, stream);
    } else {
      ensure_soa();
      launch_gather(aos.p, soa, (int)n, F_RHO, stream);
      launch_permute<double>(out, soa.rho, dd_sel.p, (int)m, stream);
    }
    launched();
    CK(cudaStreamSynchronize(stream));
    return m;
  }
  void dd_import_rho(const uint8_t *col_mask, const double *in, int64_t m) {
    if (n == 0 && m == 0) return;
    make_soa_current();
    const int64_t k = dd_select(col_mask, false);
    if (k != m) throw ArgError{"import count does not match the selected particles"};
    launch_scatter_idx(soa.rho, in, dd_sel.p, (int)m, stream);
    launched();
    if (!soa_ahead) { // keep the AoS copy coherent too
      launch_scatter(aos.p, soa, (int)n, F_RHO, stream);
      launched();
    }
    CK(cudaStreamSynchronize(stream));
  }

  // Halo payload (x, v_pred, m, p, c: 7 doubles) + all-ranks of the selected particles.
  int64_t dd_export_halo(const uint8_t *col_mask, double *out, long long *ranks_out, int64_t cap) {
    if (n == 0) return 0;
    make_soa_current();
    const int64_t m = dd_select(col_mask, false);
    if (m > cap) throw ArgError{"export buffer too small"};
    launch_export_halo(out, soa, dd_sel.p, (int)m, stream);
    if (ranks_out) launch_permute<long long>(ranks_out, all_rank.p, dd_sel.p, (int)m, stream);
    launched(2);
    CK(cudaStreamSynchronize(stream));
    return m;
  }
  // Halo particles appended from their payload: SoA fields (the rest zero), zero record tails.
  void dd_append_halo(const double *in, const long long *ranks, int64_t m) {
    if (m <= 0) return;
    normalize_tails();
    if (n + m >= (1LL << 31)) throw ArgError{"particle count out of range"};
    make_soa_current();
    soa_ahead = true; // the appended particles exist in the SoA mirror only
    grow_state(n + m);
    CK(cudaMemsetAsync(aos.p + n, 0, sizeof(Particle) * m, stream));
    CK(cudaMemcpyAsync(all_rank.p + n, ranks, sizeof(long long) * m, cudaMemcpyDeviceToDevice, stream));
    launch_append_halo(soa_at(n), in, (int)m, stream);
    launched();
    n += m;
    fixup_ok = false;
    alloc_for(n, ncells);
    dd_reset_host_order();
    need_rebin = true;
    CK(cudaStreamSynchronize(stream));
  }

  // Force on the owned cells with cell_mask[c] set (the halo-independent interior while the
  // halo rho is in flight, then the rest): a work list of those cells only.
  void force_cells(const Params &par, const uint8_t *cell_mask, int path) {
    sub_mask.ensure(ncells);
    sub_cnt.ensure(ncells);
    items_sub.ensure((size_t)ncells + (size_t)n / kTI + 1);
    CK(cudaMemcpyAsync(sub_mask.p, cell_mask, ncells, cudaMemcpyHostToDevice, stream));
    launch_subset_counts(sub_cnt.p, cnt.p, sub_mask.p, ncells, stream);
    launch_make_items(items_sub.p, scalars.p, pairs_dev.p, sub_cnt.p, cell_begin.p, na_cell.p,
                      cell_order.p, ncells, stream, kTI, items_scratch());
    launched(2);
    CK(cudaMemcpyAsync(h_small.p, scalars.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    const int ni = *(int *)h_small.p;
    sweep(SPH_FORCE, par, path, items_sub.p, ni);
  }

  // One sweep on the device. Events: ev[0..3] bracket prologue / compute / epilogue.
  void sweep(int kernel, const Params &par, int path, const Item *f_items = nullptr,
             int f_nitems = -1) {
    if (need_rebin && (kernel == SPH_DENSITY || kernel == SPH_FORCE))
      throw ArgError{"particles were appended: call sph_rebin before a pair sweep"};
    const int mode = mode_for(path);
    const bool exact = numerics == SPH_NUMERICS_EXACT;
    if (mode == SPH_LAYOUT_RESIDENT) {
      make_soa_current();
    } else {
      make_aos_current();
      if (mode == SPH_LAYOUT_CONVERT) ensure_soa();
    }
    CK(cudaEventRecord(ev[0], stream));
    if (mode == SPH_LAYOUT_CONVERT) {
      launch_gather(aos.p, soa, (int)n, kernel_in(kernel), stream); // AoS -> SoA view
      launched();
    }
    CK(cudaEventRecord(ev[1], stream));
    const bool use_aos = mode == SPH_LAYOUT_AOS;
    if (kernel == SPH_DENSITY) run_density(use_aos, exact, par, false);
    else if (kernel == SPH_FORCE) run_force(use_aos, exact, par, f_items, f_nitems);
    else {
      launch_linear(kernel, use_aos, aos.p, soa, (int)n, par, stream);
      launched();
    }
    CK(cudaEventRecord(ev[2], stream));
    if (mode == SPH_LAYOUT_CONVERT) {
      launch_scatter(aos.p, soa, (int)n, kernel_out(kernel), stream); // SoA -> AoS (Out/InOut)
      launched();
    }
    CK(cudaEventRecord(ev[3], stream));
    if (mode == SPH_LAYOUT_RESIDENT) soa_ahead = true;
    else soa_valid = false;
    dirty |= kernel_out(kernel);
  }

  // ---- host <-> device ----
  // recs[k] == recs[0] + k * 272 for every k (one flat record array in bound order)
  bool contiguous(void *const *recs) const {
    if (n <= 0) return true;
    const char *b = static_cast<const char *>(recs[0]);
    std::atomic<bool> ok{true};
    parallel_for(n, [&](int64_t lo, int64_t hi) {
      for (int64_t k = lo; k < hi; ++k)
        if (static_cast<const char *>(recs[k]) != b + k * SPH_RECORD_SIZE) {
          ok = false;
          return;
        }
    });
    return ok;
  }

  // upload_full for the end-to-end step, with the contiguity check overlapped with the
  // copy: the pointer list is verified in slices, and each verified slice of the flat record
  // array is put on the copy queue at once, so only the first slice's check is exposed (a
  // whole-list check costs ~1-2 ms of host time at 2^21 records before any byte moves).
  // Returns whether the records were one flat array; if not, the staged path redoes the
  // upload (the slices already queued read verified records only).
  bool upload_full_checked(void *const *recs) {
    if (n == 0) return true;
    const size_t bytes = (size_t)n * SPH_RECORD_SIZE;
    const char *b = static_cast<const char *>(recs[0]);
    char *dst;
    if (identity_order) {
      dst = reinterpret_cast<char *>(aos.p);
    } else {
      dense.ensure(bytes);
      dst = static_cast<char *>(dense.p);
    }
    // slices of 2^14, 2^16, then 2^18 records (~71 MB, ~1.3 ms of copy): a pointer check
    // (~1 ns per record) stays ahead of the copy (~5 ns per record) from the second slice on
    int64_t slice = 1 << 14;
    for (int64_t s = 0, e; s < n; s = e, slice = std::min<int64_t>(slice * 4, 1 << 18)) {
      e = std::min<int64_t>(n, s + slice);
      for (int64_t k = s; k < e; ++k)
        if (static_cast<const char *>(recs[k]) != b + k * SPH_RECORD_SIZE) {
          upload_full(recs, 0);
          return false;
        }
      CK(cudaMemcpyAsync(dst + s * SPH_RECORD_SIZE, b + s * SPH_RECORD_SIZE,
                         (size_t)(e - s) * SPH_RECORD_SIZE, cudaMemcpyHostToDevice, stream));
    }
    if (!identity_order) {
      launch_expand(aos.p, reinterpret_cast<Particle *>(dense.p), host_idx.p, (int)n, stream);
      launched();
    }
    soa_valid = false;
    soa_ahead = false;
    home_on = false; // whole records, slot order
    dirty = 0;
    return true;
  }

  // Full records, bound order -> device slots.
  void upload_full(void *const *recs, int contig = -1) {
    const size_t bytes = (size_t)n * SPH_RECORD_SIZE;
    if (n == 0) return;
    if (contig < 0) { // unknown: check while copying
      upload_full_checked(recs);
      return;
    }
    const void *src;
    if (contig) {
      src = recs[0];
    } else {
      h_stage.ensure(bytes);
      char *st = static_cast<char *>(h_stage.p);
      parallel_for(n, [&](int64_t b, int64_t e) {
        for (int64_t k = b; k < e; ++k) std::memcpy(st + k * SPH_RECORD_SIZE, recs[k], SPH_RECORD_SIZE);
      });
      src = h_stage.p;
    }
    if (identity_order) {
      CK(cudaMemcpyAsync(aos.p, src, bytes, cudaMemcpyHostToDevice, stream));
    } else {
      dense.ensure(bytes);
      CK(cudaMemcpyAsync(dense.p, src, bytes, cudaMemcpyHostToDevice, stream));
      launch_expand(aos.p, reinterpret_cast<Particle *>(dense.p), host_idx.p, (int)n, stream);
      launched();
    }
    soa_valid = false;
    soa_ahead = false;
    home_on = false; // whole records, slot order
    dirty = 0;
  }

  // Fields in `mask`, bound order -> device slots (AoS). Returns H2D bytes.
  size_t upload_fields(void *const *recs, uint32_t mask);

  // Device -> host: the fields in `mask` (default: dirty). Returns D2H bytes.
  size_t download_fields(void *const *recs, uint32_t mask) {
    if (n == 0 || !mask) return 0;
    make_aos_current();
    const size_t bytes = packed_bytes(mask, (size_t)n);
    dense.ensure(bytes);
    h_stage.ensure(bytes);
    launch_pack(dense.p, aos.p, host_idx.p, (int)n, mask, stream);
    launched();
    CK(cudaMemcpyAsync(h_stage.p, dense.p, bytes, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    const char *st = static_cast<const char *>(h_stage.p);
    // per-field blocks, ascending field order (pack_kernel layout)
    std::vector<std::pair<HostField, size_t>> fl;
    size_t base = 0;
    for (const HostField &f : kHostFields)
      if (mask & f.bit) {
        fl.push_back({f, base});
        base += ((size_t)f.size * (size_t)n + 15) & ~(size_t)15;
      }
    parallel_for(n, [&](int64_t b, int64_t e) {
      for (int64_t k = b; k < e; ++k) {
        char *rec = static_cast<char *>(recs[k]);
        for (auto &pf : fl)
          std::memcpy(rec + pf.first.offset, st + pf.second + (size_t)k * pf.first.size, pf.first.size);
      }
    });
    return bytes;
  }

  void download_all(void *const *recs) {
    if (n == 0) return;
    make_aos_current();
    const size_t bytes = (size_t)n * SPH_RECORD_SIZE;
    if (!identity_order) { // device work first: the host's pointer-list check overlaps it
      dense.ensure(bytes);
      launch_compact(reinterpret_cast<Particle *>(dense.p), aos.p, host_idx.p, (int)n, stream);
      launched();
    }
    const bool contig = contiguous(recs);
    void *dst = contig ? recs[0] : (h_stage.ensure(bytes), h_stage.p);
    CK(cudaMemcpyAsync(dst, identity_order ? static_cast<void *>(aos.p) : dense.p, bytes,
                       cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    if (!contig) {
      const char *st = static_cast<const char *>(h_stage.p);
      parallel_for(n, [&](int64_t b, int64_t e) {
        for (int64_t k = b; k < e; ++k) std::memcpy(recs[k], st + k * SPH_RECORD_SIZE, SPH_RECORD_SIZE);
      });
    }
    dirty = 0;
  }

  void bind(void *const *recs, const int64_t *cb64, int nx_, int ny_, double cs,
            const int64_t *rank) {
    if (nx_ <= 0 || ny_ <= 0) throw ArgError{"nx and ny must be positive"};
    const int nc = nx_ * ny_;
    const int64_t nn = cb64[nc];
    if (nn < 0 || nn >= (1LL << 31)) throw ArgError{"particle count out of range"};
    if (cb64[0] != 0) throw ArgError{"cell_begin[0] must be 0"};
    std::vector<int> cb(nc + 1);
    for (int c = 0; c <= nc; ++c) {
      if (c > 0 && cb64[c] < cb64[c - 1]) throw ArgError{"cell_begin must be non-decreasing"};
      cb[c] = (int)cb64[c];
    }
    for (int64_t k = 0; k < nn; ++k)
      if (!recs[k]) throw ArgError{"null record pointer"};
    n = nn;
    nx = nx_;
    ny = ny_;
    ncells = nc;
    cell_size = cs;
    alloc_for(n, nc);
    soa_valid = false;
    soa_ahead = false;
    identity_order = true;
    fixup_ok = false; // the first rebin sorts (the caller's in-cell order is not assumed)
    CK(cudaMemcpyAsync(cell_begin.p, cb.data(), sizeof(int) * (nc + 1), cudaMemcpyHostToDevice, stream));
    std::vector<int> hid(std::max<int64_t>(n, 1));
    std::vector<long long> ar(std::max<int64_t>(n, 1));
    for (int64_t k = 0; k < n; ++k) {
      hid[k] = (int)k;
      ar[k] = rank ? (long long)rank[k] : (long long)k;
    }
    CK(cudaMemcpyAsync(host_idx.p, hid.data(), sizeof(int) * n, cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(all_rank.p, ar.data(), sizeof(long long) * n, cudaMemcpyHostToDevice, stream));
    upload_full(recs);
    rebuild_worklist();
    sync_items0(); // (host vectors above stay alive until here)
    bound = true;
    stats = sph_stats{};
    stats.n = n;
    stats.nx = nx;
    stats.ny = ny;
    stats.ncells = ncells;
    stats.active_pairs = active_pairs;
  }

  // Permute every per-particle mirror: new slot k <- old slot perm[k], k < m (m may be
  // smaller than n: the dropped slots vanish). AoS, host_idx, all_rank, and the SoA arrays
  // when they hold data.
  void apply_perm(const int *perm, int64_t m) {
    normalize_tails();
    aos_tmp.ensure(m);
    if (soa_ahead) // the SoA is the truth: move only the AoS-only fields
      launch_permute_record_tails(aos_tmp.p, aos.p, perm, (int)m, stream);
    else
      launch_permute<Particle>(aos_tmp.p, aos.p, perm, (int)m, stream);
    std::swap(aos.p, aos_tmp.p);
    std::swap(aos.cap, aos_tmp.cap);
    host_idx_tmp.ensure(m);
    launch_permute<int>(host_idx_tmp.p, host_idx.p, perm, (int)m, stream);
    std::swap(host_idx.p, host_idx_tmp.p);
    std::swap(host_idx.cap, host_idx_tmp.cap);
    all_rank_tmp.ensure(m);
    launch_permute<long long>(all_rank_tmp.p, all_rank.p, perm, (int)m, stream);
    std::swap(all_rank.p, all_rank_tmp.p);
    std::swap(all_rank.cap, all_rank_tmp.cap);
    launched(4);
    if (soa_valid || soa_ahead) {
      auto p2 = [&](DevBuf<double2> &b) {
        tmp2.ensure(m);
        launch_permute<double2>(tmp2.p, b.p, perm, (int)m, stream);
        std::swap(b.p, tmp2.p);
        std::swap(b.cap, tmp2.cap);
        launched();
      };
      auto p1 = [&](DevBuf<double> &b) {
        tmp1.ensure(m);
        launch_permute<double>(tmp1.p, b.p, perm, (int)m, stream);
        std::swap(b.p, tmp1.p);
        std::swap(b.cap, tmp1.cap);
        launched();
      };
      p2(f_x); p2(f_v); p2(f_vp); p2(f_a);
      p1(f_m); p1(f_rho); p1(f_p); p1(f_u); p1(f_upred); p1(f_udt); p1(f_c); p1(f_h);
      p1(f_wc); p1(f_rdh); p1(f_rot); p1(f_div); p1(f_vsig); p1(f_hdt); p1(f_dtn); p1(f_dbg0);
      {
        // frozen / moved (int32) and flags (int64) through the scratch int / int64 buffers
        vals.ensure(m);
        launch_permute<int>(vals.p, f_frozen.p, perm, (int)m, stream);
        std::swap(f_frozen.p, vals.p);
        std::swap(f_frozen.cap, vals.cap);
        launch_permute<int>(vals.p, f_moved.p, perm, (int)m, stream);
        std::swap(f_moved.p, vals.p);
        std::swap(f_moved.cap, vals.cap);
        tmp8.ensure(m);
        launch_permute<int64_t>(tmp8.p, f_flags.p, perm, (int)m, stream);
        std::swap(f_flags.p, tmp8.p);
        std::swap(f_flags.cap, tmp8.cap);
        launched(3);
      }
      soa = SoaMirror{f_x.p, f_v.p, f_vp.p, f_a.p, f_m.p, f_rho.p, f_p.p, f_u.p, f_upred.p,
                      f_udt.p, f_c.p, f_h.p, f_wc.p, f_rdh.p, f_rot.p, f_div.p, f_vsig.p,
                      f_hdt.p, f_dtn.p, f_dbg0.p, f_frozen.p, f_moved.p, f_flags.p};
    }
  }

  // build_grid (grid.cpp:145-184) after a drift, by fix-up: the slots are already in
  // (cell, all_rank) order from the last rebin, only the movers change cell and the stayers
  // keep their order, so the new order is a per-cell merge (kernels_layout.cu fixup_*), and
  // every per-slot array moves in one fused pass. Same result as the sort, byte for byte.
  void rebin_fixup(bool in_step) {
    const int N = (int)n;
    slot_cell_tmp.ensure(n); fx_moved.ensure(n + 1); fx_mpos.ensure(n + 1); fx_inlist.ensure(n);
    fx_perm.ensure(n); cellnew.ensure(n);
    fx_out.ensure(ncells); fx_in.ensure(ncells); fx_in_begin.ensure(ncells);
    fx_in_fill.ensure(ncells); fx_new_begin.ensure(ncells + 1);
    const size_t sb = fixup_scan_bytes(N);
    fx_scan.ensure(sb);
    FixupArgs F{};
    F.n = N; F.ncells = ncells; F.nx = nx; F.ny = ny;
    F.aos = aos.p; F.soa = soa; F.aos_src = !soa_ahead;
    F.slot_cell = slot_cell.p; F.cell_begin = cell_begin.p; F.all_rank = all_rank.p;
    F.cellnew = cellnew.p; F.moved = fx_moved.p; F.mpos = fx_mpos.p; F.out_cnt = fx_out.p;
    F.in_cnt = fx_in.p; F.in_begin = fx_in_begin.p; F.in_fill = fx_in_fill.p;
    F.inlist = fx_inlist.p; F.new_begin = fx_new_begin.p; F.perm = fx_perm.p;
    F.scan_tmp = fx_scan.p; F.scan_bytes = sb;
    launch_rebin_fixup(F, stream);
    launched(6);
    // the SoA mirror moves only when it is the truth (resident); an AoS-side copy is dropped
    const bool soa_data = soa_ahead;
    if (!soa_ahead) soa_valid = false;
    SoaMirror dst{};
    if (soa_data) {
      const size_t M = (size_t)n;
      g_x.ensure(M); g_v.ensure(M); g_vp.ensure(M); g_a.ensure(M); g_m.ensure(M);
      g_rho.ensure(M); g_p.ensure(M); g_u.ensure(M); g_upred.ensure(M); g_udt.ensure(M);
      g_c.ensure(M); g_h.ensure(M); g_wc.ensure(M); g_rdh.ensure(M); g_rot.ensure(M);
      g_div.ensure(M); g_vsig.ensure(M); g_hdt.ensure(M); g_dtn.ensure(M); g_dbg0.ensure(M);
      g_frozen.ensure(M); g_moved.ensure(M); g_flags.ensure(M);
      dst = SoaMirror{g_x.p, g_v.p, g_vp.p, g_a.p, g_m.p, g_rho.p, g_p.p, g_u.p, g_upred.p,
                      g_udt.p, g_c.p, g_h.p, g_wc.p, g_rdh.p, g_rot.p, g_div.p, g_vsig.p,
                      g_hdt.p, g_dtn.p, g_dbg0.p, g_frozen.p, g_moved.p, g_flags.p};
    }
    host_idx_tmp.ensure(n);
    all_rank_tmp.ensure(n);
    auto sw = [](auto &a, auto &b) { std::swap(a.p, b.p); std::swap(a.cap, b.cap); };
    // resident (SoA ahead): the record fields without a SoA array stay in place and the
    // slot -> record map moves instead (a mover's p->cell written where it lives);
    // otherwise whole records move, then p->cell
    if (soa_ahead) {
      home.ensure(n);
      home_tmp.ensure(n);
    }
    launch_permute_fused(fx_perm.p, N, soa, dst, soa_data, host_idx.p, host_idx_tmp.p,
                         all_rank.p, all_rank_tmp.p, cellnew.p, slot_cell_tmp.p, slot_cell.p,
                         soa_ahead && home_on ? home.p : nullptr,
                         soa_ahead ? home_tmp.p : nullptr, aos.p, in_step, stream);
    launched();
    if (soa_ahead) {
      sw(home, home_tmp);
      home_on = true;
    } else {
      aos_tmp.ensure(n);
      launch_permute<Particle>(aos_tmp.p, aos.p, fx_perm.p, N, stream);
      launched();
      sw(aos, aos_tmp);
    }
    sw(host_idx, host_idx_tmp); sw(all_rank, all_rank_tmp);
    sw(slot_cell, slot_cell_tmp); sw(cell_begin, fx_new_begin);
    if (soa_data) {
      sw(f_x, g_x); sw(f_v, g_v); sw(f_vp, g_vp); sw(f_a, g_a); sw(f_m, g_m); sw(f_rho, g_rho);
      sw(f_p, g_p); sw(f_u, g_u); sw(f_upred, g_upred); sw(f_udt, g_udt); sw(f_c, g_c);
      sw(f_h, g_h); sw(f_wc, g_wc); sw(f_rdh, g_rdh); sw(f_rot, g_rot); sw(f_div, g_div);
      sw(f_vsig, g_vsig); sw(f_hdt, g_hdt); sw(f_dtn, g_dtn); sw(f_dbg0, g_dbg0);
      sw(f_frozen, g_frozen); sw(f_moved, g_moved); sw(f_flags, g_flags);
      soa = SoaMirror{f_x.p, f_v.p, f_vp.p, f_a.p, f_m.p, f_rho.p, f_p.p, f_u.p, f_upred.p,
                      f_udt.p, f_c.p, f_h.p, f_wc.p, f_rdh.p, f_rot.p, f_div.p, f_vsig.p,
                      f_hdt.p, f_dtn.p, f_dbg0.p, f_frozen.p, f_moved.p, f_flags.p};
    }
    if (!soa_ahead) {
      launch_set_cell(aos.p, cell_begin.p, ncells, stream); // build_grid writes p->cell
      launched();
    }
    dirty |= F_CELL;
    identity_order = false;
    rebuild_worklist();
  }

  // in_step: called between drift and density by sph_step / sph_step_host
  void rebin(bool in_step = false) {
    if (n == 0) return;
    need_rebin = false;
    if (fixup_ok && rebin_fixup_on) {
      rebin_fixup(in_step);
      return;
    }
    const bool soa_src = soa_ahead;
    keys.ensure(n); keys_sorted.ensure(n); vals.ensure(n); vals_sorted.ensure(n); cellnew.ensure(n);
    launch_rebin_keys(keys.p, vals.p, cellnew.p, aos.p, soa, !soa_src, all_rank.p, (int)n, nx, ny, stream);
    launched();
    int end_bit = 40;
    while ((1LL << (end_bit - 40)) < ncells) ++end_bit;
    size_t tmp_bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.p, keys_sorted.p, vals.p,
                                       vals_sorted.p, (int)n, 0, end_bit, stream));
    cub_tmp.ensure(tmp_bytes);
    CK(cub::DeviceRadixSort::SortPairs(cub_tmp.p, tmp_bytes, keys.p, keys_sorted.p, vals.p,
                                       vals_sorted.p, (int)n, 0, end_bit, stream));
    launched(4);
    const int *perm = vals_sorted.p;
    launch_cell_begin_from_sorted(cell_begin.p, keys_sorted.p, (int)n, ncells, stream);
    apply_perm(perm, n);
    launch_set_cell(aos.p, cell_begin.p, ncells, stream); // build_grid writes p->cell (grid.cpp:156)
    slot_cell.ensure(n);
    launch_slot_cell_from_keys(slot_cell.p, keys_sorted.p, (int)n, stream);
    launched(2);
    fixup_ok = true;
    dirty |= F_CELL;
    identity_order = false;
    rebuild_worklist();
  }
};

size_t sph_ctx::upload_fields(void *const *recs, uint32_t mask) {
  if (n == 0 || !mask) return 0;
  make_aos_current();
  // host pack: per-field blocks in bound order, then device unpack into slots
  std::vector<std::pair<HostField, size_t>> fl;
  size_t base = 0;
  for (const HostField &f : kHostFields)
    if (mask & f.bit) {
      fl.push_back({f, base});
      base += ((size_t)f.size * (size_t)n + 15) & ~(size_t)15;
    }
  h_stage.ensure(base);
  char *st = static_cast<char *>(h_stage.p);
  parallel_for(n, [&](int64_t b, int64_t e) {
    for (int64_t k = b; k < e; ++k) {
      const char *rec = static_cast<const char *>(recs[k]);
      for (auto &pf : fl)
        std::memcpy(st + pf.second + (size_t)k * pf.first.size, rec + pf.first.offset, pf.first.size);
    }
  });
  dense.ensure(base);
  CK(cudaMemcpyAsync(dense.p, st, base, cudaMemcpyHostToDevice, stream));
  launch_unpack_fields(aos.p, dense.p, host_idx.p, (int)n, mask, stream);
  launched();
  soa_valid = false;
  return base;
}

// ---------------------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------------------
namespace {
template <class F> int guarded(sph_ctx *ctx, F &&fn) {
  if (!ctx) return SPH_E_ARG;
  try {
    CK(cudaSetDevice(ctx->device));
    int r = fn();
    if (r == SPH_OK) ctx->err.clear();
    return r;
  } catch (const CudaError &e) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "CUDA error %s (%s) in %s [capi.cu:%d]", cudaGetErrorName(e.e),
                  cudaGetErrorString(e.e), e.what, e.line);
    ctx->err = buf;
    cudaGetLastError();
    return SPH_E_CUDA;
  } catch (const ArgError &e) {
    ctx->err = e.msg;
    return SPH_E_ARG;
  } catch (const std::bad_alloc &) {
    ctx->err = "host out of memory";
    return SPH_E_CUDA;
  }
}

Params to_params(const sph_params *p) {
  return Params{p->dt, p->gamma, p->cfl, p->grav, p->target_wcount};
}

void check_kernel(int k) {
  if (k < SPH_DENSITY || k > SPH_KICK2) throw ArgError{"unknown kernel id"};
}
} // namespace

extern "C" {

int sph_abi_version(void) { return SPH_B200_ABI_VERSION; }

int sph_create(int device, sph_ctx **out) {
  if (!out) return SPH_E_ARG;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0) {
    cudaGetLastError();
    return SPH_E_CUDA;
  }
  if (device < 0 || device >= ndev) return SPH_E_ARG;
  sph_ctx *ctx = new (std::nothrow) sph_ctx;
  if (!ctx) return SPH_E_CUDA;
  ctx->device = device;
  if (const char *e = std::getenv("SPH_B200_CULL")) ctx->cull = std::atoi(e) != 0;
  if (const char *e = std::getenv("SPH_B200_DEV_ROUNDS")) ctx->dev_rounds = std::atoi(e) != 0;
  if (const char *e = std::getenv("SPH_B200_PERSIST0")) ctx->persist0 = std::atoi(e) != 0;
  if (const char *e = std::getenv("SPH_B200_F2_PERSIST")) ctx->f2_persist = std::atoi(e) != 0;
  if (const char *e = std::getenv("SPH_B200_REBIN_FIXUP")) ctx->rebin_fixup_on = std::atoi(e);
  if (const char *e = std::getenv("SPH_B200_FORCE2")) ctx->force2 = std::atoi(e);
  if (const char *e = std::getenv("SPH_B200_PIPELINE")) ctx->pipeline = std::atoi(e);
  if (const char *e = std::getenv("SPH_B200_PIPE_K"))
    ctx->pipe_k = std::min(sph_ctx::kMaxPipeK, std::max(2, std::atoi(e)));
  if (const char *e = std::getenv("SPH_B200_PIPE_TAIL")) ctx->pipe_tail = std::max(1, std::atoi(e));
  if (const char *e = std::getenv("SPH_B200_DEN_JS0")) ctx->den_js0 = std::atoi(e);
  if (const char *e = std::getenv("SPH_B200_DEN_JS1")) ctx->den_js1 = std::atoi(e);
  if (const char *e = std::getenv("SPH_B200_DEN_DENSE")) ctx->den_dense_frac = std::atof(e);
  if (const char *e = std::getenv("SPH_B200_DEN_DENSE_ABS")) ctx->den_dense_abs = std::atoi(e);
  int r = guarded(ctx, [&] {
    CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    ctx->own_stream = ctx->stream;
    for (auto &e : ctx->ev) CK(cudaEventCreate(&e));
    for (auto &e : ctx->rev) CK(cudaEventCreate(&e));
    return SPH_OK;
  });
  if (r != SPH_OK) {
    delete ctx;
    return r;
  }
  *out = ctx;
  return SPH_OK;
}

void sph_destroy(sph_ctx *ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  delete ctx;
}

const char *sph_last_error(const sph_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int sph_set_numerics(sph_ctx *ctx, int numerics) {
  return guarded(ctx, [&] {
    if (numerics != SPH_NUMERICS_EXACT && numerics != SPH_NUMERICS_FAST) throw ArgError{"bad numerics"};
    ctx->numerics = numerics;
    ctx->stats.numerics = numerics;
    return SPH_OK;
  });
}

int sph_set_layout(sph_ctx *ctx, int layout) {
  return guarded(ctx, [&] {
    if (layout < SPH_LAYOUT_FROM_PATH || layout > SPH_LAYOUT_RESIDENT) throw ArgError{"bad layout"};
    ctx->layout = layout;
    ctx->stats.layout = layout;
    return SPH_OK;
  });
}

int sph_bind(sph_ctx *ctx, void *const *recs, const int64_t *cell_begin, int nx, int ny,
             double cell_size, const int64_t *all_rank) {
  return guarded(ctx, [&] {
    if (!cell_begin) throw ArgError{"null argument"};
    if (nx <= 0 || ny <= 0 || (int64_t)nx * ny > (int64_t)INT32_MAX / 2)
      throw ArgError{"nx and ny must be positive and nx * ny must fit in an int"};
    if (!recs && cell_begin[(size_t)nx * ny] > 0) throw ArgError{"null argument"};
    ctx->bind(recs, cell_begin, nx, ny, cell_size, all_rank);
    return SPH_OK;
  });
}

int sph_set_owned_cells(sph_ctx *ctx, const uint8_t *owned) {
  return guarded(ctx, [&] {
    if (!ctx->bound) throw ArgError{"sph_set_owned_cells before sph_bind"};
    if (owned) {
      ctx->owned.ensure(ctx->ncells);
      CK(cudaMemcpyAsync(ctx->owned.p, owned, ctx->ncells, cudaMemcpyHostToDevice, ctx->stream));
      ctx->has_owned = true;
    } else {
      ctx->has_owned = false;
    }
    ctx->rebuild_worklist();
    return SPH_OK;
  });
}

int sph_upload(sph_ctx *ctx, void *const *recs) {
  return guarded(ctx, [&] {
    if (!ctx->bound) throw ArgError{"sph_upload before sph_bind"};
    ctx->upload_full(recs);
    CK(cudaStreamSynchronize(ctx->stream));
    return SPH_OK;
  });
}

int sph_download(sph_ctx *ctx, void *const *recs) {
  return guarded(ctx, [&] {
    if (!ctx->bound) throw ArgError{"sph_download before sph_bind"};
    ctx->download_fields(recs, ctx->dirty);
    ctx->dirty = 0;
    return SPH_OK;
  });
}

int sph_download_all(sph_ctx *ctx, void *const *recs) {
  return guarded(ctx, [&] {
    if (!ctx->bound) throw ArgError{"sph_download_all before sph_bind"};
    ctx->download_all(recs);
    return SPH_OK;
  });
}

int sph_read_records(sph_ctx *ctx, void *out) {
  return guarded(ctx, [&] {
    if (!ctx->bound) throw ArgError{"sph_read_records before sph_bind"};
    std::vector<void *> ptrs(std::max<int64_t>(ctx->n, 1));
    for (int64_t k = 0; k < ctx->n; ++k) ptrs[k] = static_cast<char *>(out) + k * SPH_RECORD_SIZE;
    ctx->download_all(ptrs.data());
    return SPH_OK;
  });
}

int sph_sweep(sph_ctx *ctx, int kernel, const sph_params *par, int path, int order, int guard,
              sph_times *times) {
  (void)order; // LocalActive / ActiveLocal are bitwise-equivalent (test_sph.cpp:319-328)
  (void)guard; // Branch / Mask are bitwise-equivalent (test_sph.cpp:308-317)
  return guarded(ctx, [&] {
    if (!ctx->bound) throw ArgError{"sph_sweep before sph_bind"};
    if (!par) throw ArgError{"null params"};
    check_kernel(kernel);
    ctx->sweep(kernel, to_params(par), path);
    CK(cudaStreamSynchronize(ctx->stream));
    float a = 0, b = 0, c = 0;
    CK(cudaEventElapsedTime(&a, ctx->ev[0], ctx->ev[1]));
    CK(cudaEventElapsedTime(&b, ctx->ev[1], ctx->ev[2]));
    CK(cudaEventElapsedTime(&c, ctx->ev[2], ctx->ev[3]));
    if (kernel == SPH_DENSITY) ctx->stats.last_density_ms = b;
    if (kernel == SPH_FORCE) ctx->stats.last_force_ms = b;
    if (times) {
      times->prologue_ns = (int64_t)(a * 1e6);
      times->compute_ns = (int64_t)(b * 1e6);
      times->epilogue_ns = (int64_t)(c * 1e6);
    }
    return SPH_OK;
  });
}

int sph_run_sweep(sph_ctx *ctx, int kernel, void *const *recs, const sph_params *par, int path,
                  int order, int guard, sph_times *times) {
  (void)order;
  (void)guard;
  return guarded(ctx, [&] {
    if (!ctx->bound) throw ArgError{"sph_run_sweep before sph_bind"};
    if (!par) throw ArgError{"null params"};
    check_kernel(kernel);
    // Only the kernel's A_in crosses the bus on the way in and its A_out on the way back
    // (the paper's map-direction rule, "only data in A_in has to be copied").
    CK(cudaEventRecord(ctx->ev[4], ctx->stream));
    ctx->upload_fields(recs, kernel_in(kernel) | F_FLAGS);
    CK(cudaEventRecord(ctx->ev[5], ctx->stream));
    ctx->sweep(kernel, to_params(par), path);
    CK(cudaEventRecord(ctx->ev[6], ctx->stream));
    ctx->download_fields(recs, kernel_out(kernel));
    ctx->dirty = 0;
    CK(cudaEventRecord(ctx->ev[7], ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    float a = 0, b = 0, c = 0;
    CK(cudaEventElapsedTime(&a, ctx->ev[4], ctx->ev[5]));
    CK(cudaEventElapsedTime(&b, ctx->ev[5], ctx->ev[6]));
    CK(cudaEventElapsedTime(&c, ctx->ev[6], ctx->ev[7]));
    if (times) {
      times->prologue_ns = (int64_t)(a * 1e6);
      times->compute_ns = (int64_t)(b * 1e6);
      times->epilogue_ns = (int64_t)(c * 1e6);
    }
    return SPH_OK;
  });
}

int sph_rebin(sph_ctx *ctx) {
  return guarded(ctx, [&] {
    if (!ctx->bound) throw ArgError{"sph_rebin before sph_bind"};
    ctx->rebin();
    CK(cudaStreamSynchronize(ctx->stream));
    return SPH_OK;
  });
}

int sph_step(sph_ctx *ctx, const sph_params *par, double *kernel_ms) {
  return guarded(ctx, [&] {
    if (!ctx->bound) throw ArgError{"sph_step before sph_bind"};
    if (!par) throw ArgError{"null params"};
    const Params p = to_params(par);
    const int path = SPH_PATH_AOS_BASELINE;
    cudaEvent_t *e = ctx->ev + 8;
    CK(cudaEventRecord(e[0], ctx->stream));
    ctx->sweep(SPH_KICK1, p, path);
    CK(cudaEventRecord(e[1], ctx->stream));
    ctx->sweep(SPH_DRIFT, p, path);
    CK(cudaEventRecord(e[2], ctx->stream));
    ctx->rebin(true);
    CK(cudaEventRecord(e[3], ctx->stream));
    ctx->sweep(SPH_DENSITY, p, path);
    CK(cudaEventRecord(e[4], ctx->stream));
    ctx->sweep(SPH_FORCE, p, path);
    CK(cudaEventRecord(e[5], ctx->stream));
    ctx->sweep(SPH_KICK2, p, path);
    CK(cudaEventRecord(e[6], ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    float ms[6];
    for (int k = 0; k < 6; ++k) CK(cudaEventElapsedTime(&ms[k], e[k], e[k + 1]));
    ctx->stats.last_density_ms = ms[3];
    ctx->stats.last_force_ms = ms[4];
    if (kernel_ms)
      for (int k = 0; k < 6; ++k) kernel_ms[k] = ms[k];
    return SPH_OK;
  });
}

int sph_step_host(sph_ctx *ctx, void *const *recs, const sph_params *par, double *kernel_ms) {
  return guarded(ctx, [&] {
    if (!ctx->bound) throw ArgError{"sph_step_host before sph_bind"};
    if (!par || !recs) throw ArgError{"null argument"};
    const Params p = to_params(par);
    const int path = SPH_PATH_AOS_BASELINE;
    cudaEvent_t *e = ctx->ev + 6; // ev[6..14]
    CK(cudaEventRecord(e[0], ctx->stream));
    const bool contig = ctx->upload_full_checked(recs);
    CK(cudaEventRecord(e[1], ctx->stream));
    ctx->sweep(SPH_KICK1, p, path);
    CK(cudaEventRecord(e[2], ctx->stream));
    ctx->sweep(SPH_DRIFT, p, path);
    CK(cudaEventRecord(e[3], ctx->stream));
    ctx->rebin(true);
    CK(cudaEventRecord(e[4], ctx->stream));
    ctx->sweep(SPH_DENSITY, p, path);
    CK(cudaEventRecord(e[5], ctx->stream));
    float pl[2] = {0, 0};
    const bool piped = ctx->can_pipeline(contig);
    if (piped) {
      ctx->force_kick2_download_pipelined(recs[0], p, pl);
      CK(cudaEventRecord(e[6], ctx->stream));
      CK(cudaEventRecord(e[7], ctx->stream));
      CK(cudaEventRecord(e[8], ctx->stream));
    } else {
      ctx->sweep(SPH_FORCE, p, path);
      CK(cudaEventRecord(e[6], ctx->stream));
      ctx->sweep(SPH_KICK2, p, path);
      CK(cudaEventRecord(e[7], ctx->stream));
      ctx->download_all(recs); // synchronises
      CK(cudaEventRecord(e[8], ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
    float ms[8];
    for (int k = 0; k < 8; ++k) CK(cudaEventElapsedTime(&ms[k], e[k], e[k + 1]));
    if (piped) { // force chunks overlap kick2 and the copy; report the exposed tail as d2h
      ms[5] = pl[0];
      ms[6] = 0.0f;
      ms[7] = pl[1];
    }
    ctx->stats.last_density_ms = ms[4];
    ctx->stats.last_force_ms = ms[5];
    if (kernel_ms)
      for (int k = 0; k < 8; ++k) kernel_ms[k] = ms[k];
    return SPH_OK;
  });
}

int sph_apply_records(sph_ctx *ctx, int kernel, void *records, int64_t n, const sph_params *par) {
  return guarded(ctx, [&] {
    if (kernel != SPH_DRIFT && kernel != SPH_KICK1 && kernel != SPH_KICK2)
      throw ArgError{"sph_apply_records takes drift, kick1 or kick2"};
    if (!par || (n > 0 && !records)) throw ArgError{"null argument"};
    if (n < 0 || n >= (1LL << 31)) throw ArgError{"record count out of range"};
    if (n == 0) return SPH_OK;
    const size_t bytes = (size_t)n * SPH_RECORD_SIZE;
    ctx->lin_recs.ensure((size_t)n);
    CK(cudaMemcpyAsync(ctx->lin_recs.p, records, bytes, cudaMemcpyHostToDevice, ctx->stream));
    // the exact streaming kernels on the records in place (AoS); the SoA view is unused
    launch_linear(kernel, true, ctx->lin_recs.p, SoaMirror{}, (int)n, to_params(par), ctx->stream);
    ctx->launched();
    CK(cudaMemcpyAsync(records, ctx->lin_recs.p, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return SPH_OK;
  });
}

int sph_host_register(sph_ctx *ctx, void *base, uint64_t bytes) {
  return guarded(ctx, [&] {
    if (!base || !bytes) throw ArgError{"null range"};
    CK(cudaHostRegister(base, (size_t)bytes, cudaHostRegisterDefault));
    return SPH_OK;
  });
}

int sph_host_unregister(sph_ctx *ctx, void *base) {
  return guarded(ctx, [&] {
    CK(cudaHostUnregister(base));
    return SPH_OK;
  });
}

int sph_make_particles(sph_ctx *ctx, int64_t n, int ppc, uint64_t seed, sph_params *par_out) {
  return sph_make_particles_ex(ctx, n, ppc, seed, SPH_IC_UNIFORM, par_out);
}

int sph_make_particles_ex(sph_ctx *ctx, int64_t n, int ppc, uint64_t seed, int kind,
                          sph_params *par_out) {
  return guarded(ctx, [&] {
    if (ppc <= 0) throw ArgError{"ppc must be positive"};
    if (kind != SPH_IC_UNIFORM && kind != SPH_IC_CLUSTERED) throw ArgError{"unknown IC kind"};
    n = std::max<int64_t>(n, 1);
    if (n >= (1LL << 31)) throw ArgError{"n too large"};
    // proto records in id order (grid.cpp:77-98); kind 1 = clustered (see sph_b200.h)
    Mt64 rng(seed);
    const int nx = grid_nx(n, ppc);
    const double cell_size = 1.0 / nx;
    const double h_warm = 0.8 * cell_size / kSupport;
    const double sigma = 1.0 * cell_size;
    double ccx[16], ccy[16];
    if (kind == SPH_IC_CLUSTERED)
      for (int k = 0; k < 16; ++k) {
        ccx[k] = rng.unit();
        ccy[k] = rng.unit();
      }
    std::vector<Particle> proto((size_t)n);
    std::vector<int> cell((size_t)n);
    for (int64_t i = 0; i < n; ++i) {
      Particle &p = proto[(size_t)i];
      std::memset(&p, 0, sizeof p);
      if (kind == SPH_IC_CLUSTERED && i >= n / 2) {
        const int k = (int)(rng.next() % 16u);
        double gx = 0.0, gy = 0.0;
        for (int t = 0; t < 12; ++t) gx += rng.unit();
        for (int t = 0; t < 12; ++t) gy += rng.unit();
        const double x0 = ccx[k] + sigma * (gx - 6.0), x1 = ccy[k] + sigma * (gy - 6.0);
        p.x[0] = x0 - std::floor(x0);
        p.x[1] = x1 - std::floor(x1);
      } else {
        p.x[0] = rng.unit();
        p.x[1] = rng.unit();
      }
      p.v[0] = (rng.unit() * 2.0 - 1.0) * 0.05;
      p.v[1] = (rng.unit() * 2.0 - 1.0) * 0.05;
      p.v_pred[0] = p.v[0];
      p.v_pred[1] = p.v[1];
      p.u = 0.5 + rng.unit();
      p.u_pred = p.u;
      p.m = 1.0 / static_cast<double>(n);
      p.h = h_warm;
      p.dt_next = 1.0e30;
      p.id = i;
      int cx = std::max(0, std::min((int)std::floor(p.x[0] * nx), nx - 1));
      int cy = std::max(0, std::min((int)std::floor(p.x[1] * nx), nx - 1));
      cell[(size_t)i] = cy * nx + cx;
      p.cell = cell[(size_t)i]; // build_grid writes p->cell (grid.cpp:156)
    }
    // continuous store: sorted by (cell, id) (grid.cpp:117-132) == stable bucket by cell
    const int nc = nx * nx;
    std::vector<int64_t> cb((size_t)nc + 1, 0);
    for (int64_t i = 0; i < n; ++i) cb[(size_t)cell[(size_t)i] + 1]++;
    for (int c = 0; c < nc; ++c) cb[(size_t)c + 1] += cb[(size_t)c];
    std::vector<int64_t> pos(cb.begin(), cb.end() - 1);
    ctx->h_stage.ensure((size_t)n * sizeof(Particle));
    Particle *sorted = static_cast<Particle *>(ctx->h_stage.p);
    for (int64_t i = 0; i < n; ++i) sorted[pos[(size_t)cell[(size_t)i]]++] = proto[(size_t)i];
    std::vector<Particle>().swap(proto);
    std::vector<void *> ptrs((size_t)n);
    for (int64_t k = 0; k < n; ++k) ptrs[(size_t)k] = sorted + k;
    ctx->bind(ptrs.data(), cb.data(), nx, nx, cell_size, nullptr);

    const int save_num = ctx->numerics, save_layout = ctx->layout;
    ctx->numerics = SPH_NUMERICS_EXACT;
    ctx->layout = SPH_LAYOUT_AOS;
    Params p{1.0e-4, 5.0 / 3.0, 0.1, 1.0, 0.0};
    // mean_wcount (grid.cpp:31-54): per-particle sums on the device, total in list order
    ctx->wc.ensure(n);
    ctx->run_density(true, true, p, true);
    std::vector<double> wc((size_t)n);
    CK(cudaMemcpyAsync(wc.data(), ctx->wc.p, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    double total = 0.0;
    for (int64_t k = 0; k < n; ++k) total += wc[(size_t)k];
    p.target_wcount = total / static_cast<double>(n);
    ctx->sweep(SPH_DENSITY, p, SPH_PATH_AOS_BASELINE);
    launch_eos(ctx->aos.p, (int)n, p.gamma, ctx->stream); // grid.cpp:137-140
    ctx->launched();
    ctx->sweep(SPH_FORCE, p, SPH_PATH_AOS_BASELINE);
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->numerics = save_num;
    ctx->layout = save_layout;
    ctx->dirty = 0;
    if (par_out) *par_out = sph_params{p.dt, p.gamma, p.cfl, p.grav, p.target_wcount};
    return SPH_OK;
  });
}

int sph_get_stats(const sph_ctx *ctx, sph_stats *out) {
  if (!ctx || !out) return SPH_E_ARG;
  // counts that may still be in flight to the host (round-0 work list)
  int r = guarded(const_cast<sph_ctx *>(ctx), [&] {
    const_cast<sph_ctx *>(ctx)->sync_items0();
    return SPH_OK;
  });
  if (r != SPH_OK) return r;
  *out = ctx->stats;
  out->layout = ctx->layout;
  out->numerics = ctx->numerics;
  return SPH_OK;
}

int sph_synchronize(sph_ctx *ctx) {
  return guarded(ctx, [&] {
    CK(cudaStreamSynchronize(ctx->stream));
    return SPH_OK;
  });
}

int sph_pair_fractions(sph_ctx *ctx, double out[4]) {
  return guarded(ctx, [&] {
    if (!ctx->bound) throw ArgError{"sph_pair_fractions before sph_bind"};
    if (!out) throw ArgError{"null argument"};
    if (ctx->need_rebin) throw ArgError{"particles were appended: call sph_rebin first"};
    ctx->make_soa_current();
    ctx->sync_items0();
    DevBuf<unsigned long long> cnt;
    cnt.ensure(3);
    launch_pair_fractions(ctx->geom(), ctx->items0.p, ctx->n_items0, ctx->ilist.p, ctx->soa, cnt.p,
                          ctx->stream);
    ctx->launched();
    unsigned long long h[3] = {0, 0, 0};
    CK(cudaMemcpyAsync(h, cnt.p, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    cnt.release();
    const double tot = (double)ctx->active_pairs;
    for (int k = 0; k < 3; ++k) out[k] = tot > 0 ? (double)h[k] / tot : 0.0;
    out[3] = tot;
    return SPH_OK;
  });
}

int sph_fp64_peak(sph_ctx *ctx, double *tflops) {
  return guarded(ctx, [&] {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    DevBuf<double> out;
    out.ensure(1);
    const int blocks = sms * 8, iters = 4096;
    launch_fp64_probe(out.p, blocks, 64, ctx->stream); // warm-up
    float ms = 0;
    for (int t = 0; t < 3; ++t) { // best of three (a peak, not an average)
      CK(cudaEventRecord(ctx->ev[0], ctx->stream));
      launch_fp64_probe(out.p, blocks, iters, ctx->stream);
      CK(cudaEventRecord(ctx->ev[1], ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      float m = 0;
      CK(cudaEventElapsedTime(&m, ctx->ev[0], ctx->ev[1]));
      if (t == 0 || m < ms) ms = m;
    }
    ctx->launched(4);
    out.release();
    const double flops = 2.0 * 64.0 * 256.0 * (double)blocks * (double)iters;
    if (tflops) *tflops = flops / (ms * 1e-3) / 1e12;
    return SPH_OK;
  });
}

int64_t sph_launch_count(const sph_ctx *ctx) { return ctx ? ctx->launches : 0; }

int64_t sph_count(const sph_ctx *ctx) { return ctx ? ctx->n : 0; }

namespace {
void dd_check(sph_ctx *ctx, const void *mask) {
  if (!ctx->bound) throw ArgError{"decomposition call before sph_bind"};
  if (!mask) throw ArgError{"null column mask"};
}
} // namespace

int sph_dd_count(sph_ctx *ctx, const uint8_t *col_mask, int64_t *count) {
  return guarded(ctx, [&] {
    dd_check(ctx, col_mask);
    const int64_t m = ctx->n ? ctx->dd_select(col_mask, false) : 0;
    if (count) *count = m;
    return SPH_OK;
  });
}

int sph_dd_export(sph_ctx *ctx, const uint8_t *col_mask, void *dev_recs, int64_t *dev_ranks,
                  int64_t cap, int64_t *count) {
  return guarded(ctx, [&] {
    dd_check(ctx, col_mask);
    if (!dev_recs && cap > 0) throw ArgError{"null record buffer"};
    const int64_t m = ctx->dd_export(col_mask, static_cast<Particle *>(dev_recs),
                                     reinterpret_cast<long long *>(dev_ranks), cap);
    if (count) *count = m;
    return SPH_OK;
  });
}

int sph_dd_remove(sph_ctx *ctx, const uint8_t *col_mask) {
  return guarded(ctx, [&] {
    dd_check(ctx, col_mask);
    ctx->dd_remove(col_mask);
    ctx->stats.n = ctx->n;
    return SPH_OK;
  });
}

int sph_dd_append(sph_ctx *ctx, const void *dev_recs, const int64_t *dev_ranks, int64_t m) {
  return guarded(ctx, [&] {
    if (!ctx->bound) throw ArgError{"decomposition call before sph_bind"};
    if (m < 0 || (m > 0 && (!dev_recs || !dev_ranks))) throw ArgError{"bad append"};
    ctx->dd_append(static_cast<const Particle *>(dev_recs),
                   reinterpret_cast<const long long *>(dev_ranks), m);
    ctx->stats.n = ctx->n;
    return SPH_OK;
  });
}

int sph_dd_export_rho(sph_ctx *ctx, const uint8_t *col_mask, double *dev_out, int64_t cap,
                      int64_t *count) {
  return guarded(ctx, [&] {
    dd_check(ctx, col_mask);
    const int64_t m = ctx->dd_export_rho(col_mask, dev_out, cap);
    if (count) *count = m;
    return SPH_OK;
  });
}

int sph_dd_import_rho(sph_ctx *ctx, const uint8_t *col_mask, const double *dev_in, int64_t m) {
  return guarded(ctx, [&] {
    dd_check(ctx, col_mask);
    if (m > 0 && !dev_in) throw ArgError{"null rho buffer"};
    ctx->dd_import_rho(col_mask, dev_in, m);
    return SPH_OK;
  });
}

int sph_dd_export_halo(sph_ctx *ctx, const uint8_t *col_mask, double *dev_out, int64_t *dev_ranks,
                       int64_t cap, int64_t *count) {
  return guarded(ctx, [&] {
    dd_check(ctx, col_mask);
    if (!dev_out && cap > 0) throw ArgError{"null halo buffer"};
    const int64_t m = ctx->dd_export_halo(col_mask, dev_out, reinterpret_cast<long long *>(dev_ranks), cap);
    if (count) *count = m;
    return SPH_OK;
  });
}

int sph_dd_append_halo(sph_ctx *ctx, const double *dev_in, const int64_t *dev_ranks, int64_t m) {
  return guarded(ctx, [&] {
    if (!ctx->bound) throw ArgError{"decomposition call before sph_bind"};
    if (m < 0 || (m > 0 && (!dev_in || !dev_ranks))) throw ArgError{"bad halo append"};
    ctx->dd_append_halo(dev_in, reinterpret_cast<const long long *>(dev_ranks), m);
    ctx->stats.n = ctx->n;
    return SPH_OK;
  });
}

int sph_sweep_cells(sph_ctx *ctx, int kernel, const sph_params *par, const uint8_t *cell_mask) {
  return guarded(ctx, [&] {
    if (!ctx->bound) throw ArgError{"sph_sweep_cells before sph_bind"};
    if (!par || !cell_mask) throw ArgError{"null argument"};
    if (kernel != SPH_FORCE) throw ArgError{"sph_sweep_cells supports the force sweep only"};
    if (ctx->need_rebin) throw ArgError{"particles were appended: call sph_rebin before a pair sweep"};
    ctx->force_cells(to_params(par), cell_mask, SPH_PATH_AOS_BASELINE);
    CK(cudaStreamSynchronize(ctx->stream));
    float b = 0;
    CK(cudaEventElapsedTime(&b, ctx->ev[1], ctx->ev[2]));
    ctx->stats.last_force_ms = b;
    return SPH_OK;
  });
}

int sph_set_stream(sph_ctx *ctx, void *stream) {
  return guarded(ctx, [&] {
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
    return SPH_OK;
  });
}

int sph_cell_counts(sph_ctx *ctx, int64_t *out) {
  return guarded(ctx, [&] {
    if (!ctx->bound) throw ArgError{"sph_cell_counts before sph_bind"};
    if (!out) throw ArgError{"null output"};
    std::vector<int> cb(ctx->ncells + 1);
    CK(cudaMemcpyAsync(cb.data(), ctx->cell_begin.p, sizeof(int) * (ctx->ncells + 1),
                       cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int c = 0; c < ctx->ncells; ++c) out[c] = cb[c + 1] - cb[c];
    return SPH_OK;
  });
}

} // extern "C"
