// kernels_gpu.cpp — link-time drop-in for the reference's proj/src/sph/kernels.cpp.
//
// Defines every symbol proj/include/soaview/sph/kernels.hpp declares, in namespace
// soaview::sph, over the C-ABI of libsph_b200.so (include/sph_b200.h). A project that
// builds the reference's soaview_sph library with this file in place of kernels.cpp (and
// links libsph_b200.so) runs its existing callers unchanged on the B200: run_bench /
// to_csv (bench.cpp:135-233), make_particles (grid.cpp:136,141), the test suite
// (tests/test_sph.cpp) and the CLI. INTEGRATION.md §2b shows the build change.
//
//   run_sweep      kernels.hpp:45-46  -> sph_bind (when the grid's lists changed) + sph_run_sweep
//   drift_one ...  kernels.hpp:52-54  -> sph_apply_records (one record, exact kernel)
//   update_count   kernels.hpp:49     -> sum of local list sizes (host)
//   kernel_name, *_view               -> the reference's names and access sets
//
// Runtime selection (environment, read once):
//   SOAVIEW_GPU_DEVICE   CUDA device ordinal (default 0)
//   SOAVIEW_GPU_NUMERICS exact (default: byte-identical to the CPU reference) | fast
//   SOAVIEW_GPU_LAYOUT   path (default: AosBaseline -> AoS in place, SoaView -> per-call
//                        AoS->SoA conversion) | aos | convert | resident
// Errors from the device library are thrown as std::runtime_error (the reference's own
// error channel one level up, bench.cpp:139-142). There is no CPU fallback: without a
// usable GPU the first call throws.
//
// KernelTimes (device time from CUDA events, not summed per-thread CPU time): AosBaseline
// sweeps report everything as compute, as the reference's do (kernels.hpp:37-38); SoaView
// sweeps report the host->device copy of the kernel's A_in as prologue, the device sweep
// (AoS->SoA gather, kernels, SoA->AoS scatter) as compute, and the device->host copy of
// A_out as epilogue: on the GPU the bus transfer is the conversion cost the paper measures.
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "sph_b200.h"
#include "soaview/sph/kernels.hpp"

namespace soaview::sph {

namespace {

static_assert(sizeof(Particle) == SPH_RECORD_SIZE, "Particle must be the 272-byte record");

struct Device {
  sph_ctx *ctx = nullptr;
  const CellGrid *bound = nullptr;
  uint64_t sig = 0;
  std::vector<Particle *> recs;
  std::vector<int64_t> cell_begin;
  std::mutex mu; // the reference's run_sweep is callable from any thread; calls serialise

  Device() {
    int dev = 0;
    if (const char *e = std::getenv("SOAVIEW_GPU_DEVICE")) dev = std::atoi(e);
    if (sph_create(dev, &ctx) != SPH_OK || !ctx)
      throw std::runtime_error("soaview::sph (B200 drop-in): no usable CUDA device");
    int numerics = SPH_NUMERICS_EXACT, layout = SPH_LAYOUT_FROM_PATH;
    if (const char *e = std::getenv("SOAVIEW_GPU_NUMERICS"))
      numerics = std::string(e) == "fast" ? SPH_NUMERICS_FAST : SPH_NUMERICS_EXACT;
    if (const char *e = std::getenv("SOAVIEW_GPU_LAYOUT")) {
      const std::string l(e);
      layout = l == "aos" ? SPH_LAYOUT_AOS
               : l == "convert" ? SPH_LAYOUT_CONVERT
               : l == "resident" ? SPH_LAYOUT_RESIDENT
                                 : SPH_LAYOUT_FROM_PATH;
    }
    check(sph_set_numerics(ctx, numerics));
    check(sph_set_layout(ctx, layout));
  }

  void check(int rc) const {
    if (rc != SPH_OK)
      throw std::runtime_error(std::string("soaview::sph (B200 drop-in): ") + sph_last_error(ctx));
  }

  // Every pointer of every local list, in order (a grid rebuilt in place re-binds).
  static uint64_t signature(const CellGrid &g) {
    uint64_t h = 1469598103934665603ULL ^ static_cast<uint64_t>(g.nx) * 131u ^ g.ny;
    for (const auto &l : g.local) {
      h = (h ^ l.size()) * 1099511628211ULL;
      for (const Particle *p : l) h = (h ^ reinterpret_cast<uintptr_t>(p)) * 1099511628211ULL;
    }
    return h;
  }

  // The device derives each cell's active list from (nx, ny) as build_grid builds it
  // (grid.cpp:159-182: the wrapped 3x3 stencil, row-major, deduplicated); a grid whose
  // active lists are anything else is rejected rather than silently swept differently.
  static void check_stencil(const CellGrid &g) {
    if (g.nx <= 0 || g.ny <= 0 || g.local.size() != static_cast<size_t>(g.cells()) ||
        g.active.size() != g.local.size())
      throw std::runtime_error("soaview::sph (B200 drop-in): malformed CellGrid");
    for (int c = 0; c < g.cells(); ++c) {
      const int cy = c / g.nx, cx = c % g.nx;
      int seen[9], ns = 0;
      size_t pos = 0;
      const auto &act = g.active[static_cast<size_t>(c)];
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const int k = ((cy + dy + g.ny) % g.ny) * g.nx + (cx + dx + g.nx) % g.nx;
          bool dup = false;
          for (int q = 0; q < ns; ++q) dup |= seen[q] == k;
          if (dup) continue;
          seen[ns++] = k;
          for (const Particle *p : g.local[static_cast<size_t>(k)])
            if (pos >= act.size() || act[pos++] != p)
              throw std::runtime_error(
                  "soaview::sph (B200 drop-in): active lists are not the build_grid stencil");
        }
      if (pos != act.size())
        throw std::runtime_error(
            "soaview::sph (B200 drop-in): active lists are not the build_grid stencil");
    }
  }

  void bind(const CellGrid &g) {
    const uint64_t s = signature(g);
    if (bound == &g && s == sig) return;
    check_stencil(g);
    recs.clear();
    cell_begin.assign(1, 0);
    for (const auto &l : g.local) {
      recs.insert(recs.end(), l.begin(), l.end());
      cell_begin.push_back(static_cast<int64_t>(recs.size()));
    }
    check(sph_bind(ctx, reinterpret_cast<void *const *>(recs.data()), cell_begin.data(), g.nx, g.ny,
                   g.cell_size, nullptr));
    bound = &g;
    sig = s;
  }
};

// Never destroyed: tearing the context down from a static destructor could run after the
// CUDA runtime has unloaded; the process exit releases the device.
Device &device() {
  static Device *d = new Device;
  return *d;
}

sph_params cpar(const SphParams &p) { return sph_params{p.dt, p.gamma, p.cfl, p.grav, p.target_wcount}; }

// Access sets of the reference's view descriptors (kernels.cpp:741-859), one row per field in
// descriptor order: the GPU path moves exactly these bytes (sph_run_sweep uploads A_in and
// downloads A_out). 'i' In, 'o' Out, 'b' InOut.
struct Row {
  size_t off;
  int size;
  char dir;
};
#define F(name, sz, d) Row{offsetof(Particle, name), sz, d}
const std::vector<Row> kDensityLocal = {F(x, 16, 'i'),     F(v_pred, 16, 'i'), F(m, 8, 'i'),
                                        F(h, 8, 'b'),      F(rho, 8, 'b'),     F(wcount, 8, 'b'),
                                        F(rho_dh, 8, 'b'), F(rot_v, 8, 'b'),   F(div_v, 8, 'b')};
const std::vector<Row> kDensityActive = {F(x, 16, 'i'), F(v_pred, 16, 'i'), F(m, 8, 'i')};
const std::vector<Row> kForceLocal = {
    F(x, 16, 'i'),     F(v_pred, 16, 'i'), F(h, 8, 'i'),    F(p, 8, 'i'),     F(rho, 8, 'i'),
    F(rho_dh, 8, 'i'), F(c, 8, 'i'),       F(div_v, 8, 'i'), F(rot_v, 8, 'i'), F(a, 16, 'b'),
    F(u_dt, 8, 'b'),   F(v_sig, 8, 'b'),   F(h_dt, 8, 'b')};
const std::vector<Row> kForceActive = {F(x, 16, 'i'), F(v_pred, 16, 'i'), F(m, 8, 'i'),
                                       F(rho, 8, 'i'), F(p, 8, 'i'),      F(c, 8, 'i')};
const std::vector<Row> kDrift = {F(x, 16, 'b'), F(v_pred, 16, 'i'), F(frozen, 4, 'i'),
                                 F(u, 8, 'i'),  F(u_dt, 8, 'i'),    F(u_pred, 8, 'o'),
                                 F(moved, 4, 'o')};
const std::vector<Row> kKick1 = {F(v, 16, 'b'), F(a, 16, 'i'), F(u, 8, 'b'), F(u_dt, 8, 'i'),
                                 F(dt_next, 8, 'o')};
const std::vector<Row> kKick2 = {F(v, 16, 'b'),      F(a, 16, 'i'),     F(dbg, 16, 'i'),
                                 F(u, 8, 'b'),       F(u_dt, 8, 'i'),   F(u_pred, 8, 'b'),
                                 F(rho, 8, 'i'),     F(dt_next, 8, 'b'), F(h, 8, 'i'),
                                 F(v_sig, 8, 'i'),   F(c, 8, 'b'),      F(v_pred, 16, 'o'),
                                 F(p, 8, 'o'),       F(h_dt, 8, 'o')};
#undef F

ViewDescriptor view(const std::vector<Row> &rows, int64_t count) {
  ViewDescriptor d;
  d.record_size = static_cast<int>(sizeof(Particle));
  d.count = count;
  for (const Row &r : rows)
    d.fields.push_back(FieldSpec{static_cast<int>(r.off), r.size,
                                 r.dir == 'i' ? Dir::In : r.dir == 'o' ? Dir::Out : Dir::InOut});
  return d;
}

void apply_one(int kernel, Particle &p, const SphParams &par) {
  Device &d = device();
  std::lock_guard<std::mutex> lk(d.mu);
  const sph_params cp = cpar(par);
  d.check(sph_apply_records(d.ctx, kernel, &p, 1, &cp));
}

} // namespace

const char *kernel_name(KernelId k) {
  switch (k) {
  case KernelId::Density: return "density";
  case KernelId::Force: return "force";
  case KernelId::Drift: return "drift";
  case KernelId::Kick1: return "kick1";
  default: return "kick2";
  }
}

ViewDescriptor density_local_view(int64_t count) { return view(kDensityLocal, count); }
ViewDescriptor density_active_view(int64_t count) { return view(kDensityActive, count); }
ViewDescriptor force_local_view(int64_t count) { return view(kForceLocal, count); }
ViewDescriptor force_active_view(int64_t count) { return view(kForceActive, count); }
ViewDescriptor drift_view(int64_t count) { return view(kDrift, count); }
ViewDescriptor kick1_view(int64_t count) { return view(kKick1, count); }
ViewDescriptor kick2_view(int64_t count) { return view(kKick2, count); }

KernelTimes run_sweep(KernelId k, const CellGrid &grid, const SphParams &par, Path path,
                      Order order, Guard guard, int threads) {
  (void)threads; // the device schedules its own work list (one warp per cell item)
  Device &d = device();
  std::lock_guard<std::mutex> lk(d.mu);
  d.bind(grid);
  const sph_params cp = cpar(par);
  sph_times t{};
  d.check(sph_run_sweep(d.ctx, static_cast<int>(k), reinterpret_cast<void *const *>(d.recs.data()),
                        &cp, static_cast<int>(path), static_cast<int>(order),
                        static_cast<int>(guard), &t));
  KernelTimes out;
  if (path == Path::AosBaseline) {
    out.compute_ns = t.prologue_ns + t.compute_ns + t.epilogue_ns;
  } else {
    out.prologue_ns = t.prologue_ns;
    out.compute_ns = t.compute_ns;
    out.epilogue_ns = t.epilogue_ns;
  }
  return out;
}

int64_t update_count(const CellGrid &grid) {
  int64_t n = 0;
  for (const auto &l : grid.local) n += static_cast<int64_t>(l.size());
  return n;
}

void drift_one(Particle &p, const SphParams &par) { apply_one(SPH_DRIFT, p, par); }
void kick1_one(Particle &p, const SphParams &par) { apply_one(SPH_KICK1, p, par); }
void kick2_one(Particle &p, const SphParams &par) { apply_one(SPH_KICK2, p, par); }

} // namespace soaview::sph
