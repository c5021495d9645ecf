// shim_parity.cpp — TEST INFRASTRUCTURE. One binary that links the UNMODIFIED reference
// (compiled from /root/reference by oracle/Makefile) and the GPU drop-in
// (include/soaview_gpu.hpp over libsph_b200.so), and compares them through the reference's
// own API: make_particles -> build_grid -> for every kernel:
//   soaview::sph::run_sweep       (CPU reference, threads = 4)
//   soaview::sph::gpu::run_sweep  (B200, EXACT numerics)  -> must be byte-identical
//   soaview::sph::gpu::run_sweep  (B200, FAST numerics)   -> within 1e-10
// for both Path values and both store layouts. Exit code 0 = parity.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "soaview/sph/grid.hpp"
#include "soaview/sph/kernels.hpp"
#include "soaview_gpu.hpp"

using namespace soaview::sph;

static double field_err(const std::vector<Particle> &a, const std::vector<Particle> &b, KernelId k) {
  // max over particles of |a-b| / (|b| + rms) for the kernel's output fields
  auto pick = [&](const Particle &p, int f) -> double {
    switch (k) {
    case KernelId::Density: {
      const double v[6] = {p.h, p.rho, p.wcount, p.rho_dh, p.rot_v, p.div_v};
      return v[f];
    }
    case KernelId::Force: {
      const double v[5] = {p.a[0], p.a[1], p.u_dt, p.v_sig, p.h_dt};
      return v[f];
    }
    default:
      return 0.0;
    }
  };
  int nf = k == KernelId::Density ? 6 : (k == KernelId::Force ? 5 : 0);
  double worst = 0.0;
  for (int f = 0; f < nf; ++f) {
    double rms = 0.0;
    for (const Particle &p : b) rms += pick(p, f) * pick(p, f);
    rms = std::sqrt(rms / b.size());
    for (size_t i = 0; i < a.size(); ++i) {
      double d = std::fabs(pick(a[i], f) - pick(b[i], f));
      worst = std::fmax(worst, d / (std::fabs(pick(b[i], f)) + rms + 1e-300));
    }
  }
  return worst;
}

int main() {
  int failures = 0;
  const KernelId kernels[] = {KernelId::Density, KernelId::Force, KernelId::Drift, KernelId::Kick1,
                              KernelId::Kick2};
  const char *names[] = {"density", "force", "drift", "kick1", "kick2"};
  struct Case { int64_t n; int ppc; uint64_t seed; Layout layout; };
  const Case cases[] = {{4000, 64, 42, Layout::Scattered}, {30000, 1024, 7, Layout::Continuous},
                        {250, 64, 9, Layout::Continuous}};
  auto &dev = gpu::Device::instance();
  for (const Case &cs : cases) {
    InitConfig cfg;
    cfg.n = cs.n;
    cfg.ppc = cs.ppc;
    cfg.seed = cs.seed;
    cfg.layout = cs.layout;
    SphParams par;
    ParticleStore s = make_particles(cfg, par);
    CellGrid g = build_grid(s, cfg);
    const std::vector<Particle> ic = s.snapshot();
    for (int ki = 0; ki < 5; ++ki) {
      for (Path path : {Path::AosBaseline, Path::SoaView}) {
        s.restore(ic);
        run_sweep(kernels[ki], g, par, path, Order::LocalActive, Guard::Branch, 4);
        const std::vector<Particle> ref = s.snapshot();

        s.restore(ic);
        dev.set_numerics(SPH_NUMERICS_EXACT);
        gpu::run_sweep(kernels[ki], g, par, path, Order::LocalActive, Guard::Branch);
        const std::vector<Particle> ex = s.snapshot();
        bool same = std::memcmp(ex.data(), ref.data(), ref.size() * sizeof(Particle)) == 0;

        s.restore(ic);
        dev.set_numerics(SPH_NUMERICS_FAST);
        gpu::run_sweep(kernels[ki], g, par, path, Order::ActiveLocal, Guard::Mask);
        const std::vector<Particle> fa = s.snapshot();
        double err = field_err(fa, ref, kernels[ki]);
        bool fast_ok = (ki >= 2) ? std::memcmp(fa.data(), ref.data(), ref.size() * sizeof(Particle)) == 0
                                 : err <= 1e-10;
        std::printf("n=%lld ppc=%d %s %-7s exact:%s fast:%s (max rel %.2e)\n",
                    static_cast<long long>(cs.n), cs.ppc,
                    path == Path::AosBaseline ? "aos-baseline" : "soa-view    ", names[ki],
                    same ? "byte-identical" : "DIFFERS", fast_ok ? "ok" : "FAIL", err);
        failures += !same + !fast_ok;
      }
    }
  }
  // Time stepping through the shim: kick1, drift, then `grid = build_grid(...)` into the SAME
  // CellGrid object (same address, new lists: particles crossed cells), density, force,
  // kick2. The adapter must notice the changed lists and re-bind (EXACT: byte-identical).
  {
    InitConfig cfg;
    cfg.n = 3000;
    cfg.ppc = 64;
    cfg.seed = 5;
    cfg.layout = Layout::Scattered;
    SphParams par;
    ParticleStore a = make_particles(cfg, par);
    ParticleStore b = make_particles(cfg, par);
    par.dt = 2e-3; // particles cross cells within the three steps
    CellGrid ga = build_grid(a, cfg), gb = build_grid(b, cfg);
    dev.set_numerics(SPH_NUMERICS_EXACT);
    int moved = 0;
    std::vector<int64_t> cell0;
    for (const Particle *p : a.all) cell0.push_back(p->cell);
    for (int step = 0; step < 3; ++step) {
      for (KernelId k : {KernelId::Kick1, KernelId::Drift}) {
        run_sweep(k, ga, par, Path::AosBaseline, Order::LocalActive, Guard::Branch, 4);
        gpu::run_sweep(k, gb, par, Path::AosBaseline, Order::LocalActive, Guard::Branch);
      }
      ga = build_grid(a, cfg);
      gb = build_grid(b, cfg);
      for (KernelId k : {KernelId::Density, KernelId::Force, KernelId::Kick2}) {
        run_sweep(k, ga, par, Path::AosBaseline, Order::LocalActive, Guard::Branch, 4);
        gpu::run_sweep(k, gb, par, Path::AosBaseline, Order::LocalActive, Guard::Branch);
      }
    }
    for (size_t i = 0; i < a.all.size(); ++i) moved += a.all[i]->cell != cell0[i];
    const std::vector<Particle> ra = a.snapshot(), rb = b.snapshot();
    const bool same = std::memcmp(ra.data(), rb.data(), ra.size() * sizeof(Particle)) == 0;
    std::printf("3 steps, grid rebuilt in place (%d particles changed cell): %s\n", moved,
                same ? "byte-identical" : "DIFFERS");
    failures += !same + (moved == 0);
  }
  std::printf("[shim_parity] %s (%d failures)\n", failures ? "FAILED" : "passed", failures);
  return failures ? 1 : 0;
}
