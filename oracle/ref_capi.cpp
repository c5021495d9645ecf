// ref_capi.cpp — TEST INFRASTRUCTURE (oracle), not product code.
//
// A thin extern "C" wrapper over the UNMODIFIED reference SPH implementation
// (/root/reference/proj/src/sph/{grid,kernels,bench}.cpp + src/layout.cpp), compiled
// by oracle/Makefile straight from the reference tree into oracle/_ref/libsoaview_ref.so.
// It lets the Python tests and bench.py's CPU-baseline leg call the reference's own
// make_particles / build_grid / run_sweep on plain particle arrays.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
// legs may load this library, and only as the checker or the CPU baseline.
#include <chrono>
#include <cstring>
#include <memory>
#include <vector>

#include "soaview/layout.hpp"
#include "soaview/sph/bench.hpp"
#include "soaview/sph/grid.hpp"
#include "soaview/sph/kernels.hpp"
#include "soaview/sph/spline.hpp"

using namespace soaview;
using namespace soaview::sph;

namespace {
struct RefGrid {
  ParticleStore store; // `all` points into caller-owned records
  CellGrid grid;
  InitConfig cfg;
};
SphParams to_par(const double *p5) {
  SphParams p;
  p.dt = p5[0];
  p.gamma = p5[1];
  p.cfl = p5[2];
  p.grav = p5[3];
  p.target_wcount = p5[4];
  return p;
}
} // namespace

extern "C" {

int ref_record_size() { return static_cast<int>(sizeof(Particle)); }
double ref_kernel_w(double q) { return kernel_w(q); }
double ref_kernel_dw(double q) { return kernel_dw(q); }

// grid.cpp:76-143. Writes the n records in store.all order to `out` (continuous: sorted
// by (cell, id); scattered: by id) and the calibrated SphParams to par5_out.
int ref_make_particles(int64_t n, int ppc, uint64_t seed, int layout, void *out,
                       double *par5_out) {
  InitConfig cfg;
  cfg.n = n;
  cfg.ppc = ppc;
  cfg.seed = seed;
  cfg.layout = layout ? Layout::Continuous : Layout::Scattered;
  SphParams par;
  ParticleStore s = make_particles(cfg, par);
  auto *dst = static_cast<Particle *>(out);
  for (int64_t i = 0; i < s.size(); ++i) dst[i] = *s.all[static_cast<size_t>(i)];
  par5_out[0] = par.dt;
  par5_out[1] = par.gamma;
  par5_out[2] = par.cfl;
  par5_out[3] = par.grav;
  par5_out[4] = par.target_wcount;
  return 0;
}

// build_grid (grid.cpp:145-184) over caller-owned records: store.all[i] = &recs[i].
void *ref_grid_create(void *recs, int64_t n, int ppc) {
  auto *g = new RefGrid;
  g->store.layout = Layout::Continuous;
  auto *p = static_cast<Particle *>(recs);
  g->store.all.resize(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) g->store.all[static_cast<size_t>(i)] = p + i;
  g->cfg.n = n;
  g->cfg.ppc = ppc;
  g->grid = build_grid(g->store, g->cfg);
  return g;
}

// Same, but with an explicit store.all order: all[k] = &recs[order[k]].
void *ref_grid_create_ordered(void *recs, int64_t n, int ppc, const int64_t *order) {
  auto *g = new RefGrid;
  g->store.layout = Layout::Continuous;
  auto *p = static_cast<Particle *>(recs);
  g->store.all.resize(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) g->store.all[static_cast<size_t>(i)] = p + order[i];
  g->cfg.n = n;
  g->cfg.ppc = ppc;
  g->grid = build_grid(g->store, g->cfg);
  return g;
}

void ref_grid_destroy(void *h) { delete static_cast<RefGrid *>(h); }

void ref_grid_info(void *h, int *nx, int *ny, double *cell_size, int64_t *active_total) {
  auto *g = static_cast<RefGrid *>(h);
  *nx = g->grid.nx;
  *ny = g->grid.ny;
  *cell_size = g->grid.cell_size;
  int64_t t = 0;
  for (auto &a : g->grid.active) t += static_cast<int64_t>(a.size());
  *active_total = t;
}

// Local lists as CSR of record indices (index = pointer - recs base).
void ref_grid_local_csr(void *h, void *recs, int64_t *cell_begin, int64_t *local_idx) {
  auto *g = static_cast<RefGrid *>(h);
  auto *base = static_cast<Particle *>(recs);
  int64_t k = 0;
  for (int c = 0; c < g->grid.cells(); ++c) {
    cell_begin[c] = k;
    for (Particle *p : g->grid.local[static_cast<size_t>(c)]) local_idx[k++] = p - base;
  }
  cell_begin[g->grid.cells()] = k;
}

// Active lists as CSR of record indices.
void ref_grid_active_csr(void *h, void *recs, int64_t *cell_begin, int64_t *active_idx) {
  auto *g = static_cast<RefGrid *>(h);
  auto *base = static_cast<Particle *>(recs);
  int64_t k = 0;
  for (int c = 0; c < g->grid.cells(); ++c) {
    cell_begin[c] = k;
    for (Particle *p : g->grid.active[static_cast<size_t>(c)]) active_idx[k++] = p - base;
  }
  cell_begin[g->grid.cells()] = k;
}

// Keep only the cells with mask[c] != 0 (run_sweep skips nl == 0, kernels.cpp:548);
// used to time a bounded sample of a large workload.
void ref_grid_keep_cells(void *h, const uint8_t *mask) {
  auto *g = static_cast<RefGrid *>(h);
  for (int c = 0; c < g->grid.cells(); ++c)
    if (!mask[c]) g->grid.local[static_cast<size_t>(c)].clear();
}

int64_t ref_update_count(void *h) { return update_count(static_cast<RefGrid *>(h)->grid); }

// run_sweep (kernels.cpp:861-872). times4 = {prologue, compute, epilogue, wall} ns.
int ref_run_sweep(void *h, int kernel, const double *par5, int path, int order, int guard,
                  int threads, int64_t *times4) {
  auto *g = static_cast<RefGrid *>(h);
  SphParams par = to_par(par5);
  auto t0 = std::chrono::steady_clock::now();
  KernelTimes t = run_sweep(static_cast<KernelId>(kernel), g->grid, par, static_cast<Path>(path),
                            static_cast<Order>(order), static_cast<Guard>(guard), threads);
  auto t1 = std::chrono::steady_clock::now();
  if (times4) {
    times4[0] = t.prologue_ns;
    times4[1] = t.compute_ns;
    times4[2] = t.epilogue_ns;
    times4[3] = std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
  }
  return 0;
}

void ref_drift_one(void *rec, const double *par5) {
  drift_one(*static_cast<Particle *>(rec), to_par(par5));
}
void ref_kick1_one(void *rec, const double *par5) {
  kick1_one(*static_cast<Particle *>(rec), to_par(par5));
}
void ref_kick2_one(void *rec, const double *par5) {
  kick2_one(*static_cast<Particle *>(rec), to_par(par5));
}

// View descriptors (kernels.cpp:741-859): writes (offset, size, dir) triples; returns count.
int ref_view_fields(int which, int *out3, int cap) {
  ViewDescriptor d;
  switch (which) {
  case 0: d = density_local_view(0); break;
  case 1: d = density_active_view(0); break;
  case 2: d = force_local_view(0); break;
  case 3: d = force_active_view(0); break;
  case 4: d = drift_view(0); break;
  case 5: d = kick1_view(0); break;
  default: d = kick2_view(0); break;
  }
  int k = 0;
  for (const FieldSpec &f : d.fields) {
    if (k >= cap) break;
    out3[3 * k] = f.offset;
    out3[3 * k + 1] = f.size;
    out3[3 * k + 2] = static_cast<int>(f.dir);
    ++k;
  }
  return static_cast<int>(d.fields.size());
}

} // extern "C"
