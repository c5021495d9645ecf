// soaview_gpu.hpp — header-only C++ adapter: the reference's run_sweep on the B200.
//
// For code that already uses the reference API (soaview::sph, kernels.hpp:45-46):
//
//   #include "soaview/sph/kernels.hpp"   // the reference headers, unchanged
//   #include "soaview_gpu.hpp"           // this file (+ link libsph_b200.so)
//   soaview::sph::gpu::run_sweep(KernelId::Density, grid, par, Path::AosBaseline,
//                                Order::LocalActive, Guard::Branch);
//
// The function has the reference's exact signature and semantics: it mutates the
// Particle records of `grid` in place (only each kernel's A_out bytes, kernels.cpp:741-859)
// and returns KernelTimes (prologue = host->device copy of the kernel's A_in, compute =
// device time, epilogue = device->host copy of its A_out). It lives in a sibling namespace
// so the CPU reference and the GPU path can be linked into one binary and compared.
// Path selects the device layout (AosBaseline -> AoS in place, SoaView -> per-call
// AoS->SoA conversion); Order / Guard / threads do not change results (the reference's
// variants are bitwise-equivalent, test_sph.cpp:308-346). The CellGrid is flattened and
// bound once and re-bound when its lists change (an O(n) compare of the pointer lists per call).
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <vector>

#include "sph_b200.h"
#include "soaview/sph/kernels.hpp"

namespace soaview::sph::gpu {

class Device {
public:
  static Device &instance(int device = 0) {
    static Device d(device);
    return d;
  }
  sph_ctx *ctx() const { return ctx_; }

  // numerics: SPH_NUMERICS_EXACT (byte-identical to the CPU) or SPH_NUMERICS_FAST
  void set_numerics(int numerics) { check(sph_set_numerics(ctx_, numerics)); }
  void set_layout(int layout) { check(sph_set_layout(ctx_, layout)); }

  void bind(const CellGrid &g) {
    if (bound_ == &g && same_lists(g)) return;
    recs_.clear();
    cell_begin_.assign(1, 0);
    for (const auto &l : g.local) {
      for (Particle *p : l) recs_.push_back(p);
      cell_begin_.push_back(static_cast<int64_t>(recs_.size()));
    }
    // the active lists must be the reference's wrapped, deduplicated 3x3 stencil
    // (build_grid, grid.cpp:159-182); the device derives them from (nx, ny)
    for (int c = 0; c < g.cells(); ++c) {
      size_t na = 0;
      int cy = c / g.nx, cx = c % g.nx, seen[9], ns = 0;
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          int k = ((cy + dy + g.ny) % g.ny) * g.nx + (cx + dx + g.nx) % g.nx;
          bool dup = false;
          for (int q = 0; q < ns; ++q) dup |= seen[q] == k;
          if (!dup) {
            seen[ns++] = k;
            na += g.local[static_cast<size_t>(k)].size();
          }
        }
      if (na != g.active[static_cast<size_t>(c)].size())
        throw std::runtime_error("soaview::sph::gpu: active lists are not the build_grid stencil");
    }
    check(sph_bind(ctx_, reinterpret_cast<void *const *>(recs_.data()), cell_begin_.data(), g.nx,
                   g.ny, g.cell_size, nullptr));
    bound_ = &g;
  }

  void *const *records() const { return reinterpret_cast<void *const *>(recs_.data()); }

  void check(int rc) const {
    if (rc != SPH_OK) throw std::runtime_error(std::string("libsph_b200: ") + sph_last_error(ctx_));
  }

  ~Device() { sph_destroy(ctx_); }

private:
  explicit Device(int device) {
    if (sph_create(device, &ctx_) != SPH_OK || !ctx_)
      throw std::runtime_error("libsph_b200: no usable CUDA device");
  }
  // Every pointer of every local list, in order, against the bound copy: a rebuilt grid at
  // the same address whose particles swapped cells (or were reordered) behind unchanged
  // list sizes re-binds. run_sweep walks all n pointers to pack the upload anyway, so this
  // is O(n) of the same (an exact compare, not a hash).
  bool same_lists(const CellGrid &g) const {
    if (g.local.size() + 1 != cell_begin_.size()) return false;
    size_t k = 0;
    for (size_t c = 0; c < g.local.size(); ++c) {
      const auto &l = g.local[c];
      if (static_cast<int64_t>(k + l.size()) != cell_begin_[c + 1]) return false;
      for (const Particle *p : l)
        if (recs_[k++] != p) return false;
    }
    return true;
  }
  sph_ctx *ctx_ = nullptr;
  const CellGrid *bound_ = nullptr;
  std::vector<Particle *> recs_;
  std::vector<int64_t> cell_begin_;
};

// Drop-in for soaview::sph::run_sweep (kernels.hpp:45-46).
inline KernelTimes run_sweep(KernelId k, const CellGrid &grid, const SphParams &par, Path path,
                             Order order, Guard guard, int threads = 1) {
  (void)threads;
  Device &d = Device::instance();
  d.bind(grid);
  sph_params p{par.dt, par.gamma, par.cfl, par.grav, par.target_wcount};
  sph_times t{};
  d.check(sph_run_sweep(d.ctx(), static_cast<int>(k), d.records(), &p, static_cast<int>(path),
                        static_cast<int>(order), static_cast<int>(guard), &t));
  KernelTimes out;
  out.prologue_ns = t.prologue_ns;
  out.compute_ns = t.compute_ns;
  out.epilogue_ns = t.epilogue_ns;
  return out;
}

} // namespace soaview::sph::gpu
