// kernels_exact.cu — EXACT numerics: the reference's floating-point operation sequence.
//
// Compiled with --fmad=false (like the reference's -ffp-contract=off,
// proj/src/CMakeLists.txt:21-22); CUDA double sqrt and '/' are IEEE round-to-nearest and
// round() is round-half-away-from-zero like std::round, so every expression below
// produces the same bits as the CPU. With the pair skeleton's reference j order this
// makes density, force, drift, kick1 and kick2 byte-identical to run_sweep.
//
// Contents: the EXACT pair policy (density_pair / force_pair / density_step /
// density_publish / force_inv, kernels.cpp:97-202), the mean_wcount pass
// (grid.cpp:31-54), and the streaming drift / kick1 / kick2 kernels
// (kernels.cpp:305-341), which are exact in both numerics modes.
#include "pair_kernels.cuh"
#include "sph_kernels.h"

namespace sphb {

namespace {

// spline.hpp:12-25
__device__ __forceinline__ double kernel_w(double q) {
  if (q >= 2.5) return 0.0;
  double t1 = 2.5 - q;
  double acc = t1 * t1 * t1 * t1;
  if (q < 1.5) {
    double t2 = 1.5 - q;
    acc = acc - 5.0 * (t2 * t2 * t2 * t2);
  }
  if (q < 0.5) {
    double t3 = 0.5 - q;
    acc = acc + 10.0 * (t3 * t3 * t3 * t3);
  }
  return kNorm2d * acc;
}

// spline.hpp:28-41
__device__ __forceinline__ double kernel_dw(double q) {
  if (q >= 2.5) return 0.0;
  double t1 = 2.5 - q;
  double acc = t1 * t1 * t1;
  if (q < 1.5) {
    double t2 = 1.5 - q;
    acc = acc - 5.0 * (t2 * t2 * t2);
  }
  if (q < 0.5) {
    double t3 = 0.5 - q;
    acc = acc + 10.0 * (t3 * t3 * t3);
  }
  return kNorm2d * -4.0 * acc;
}

__device__ __forceinline__ double min_image(double d) { return d - round(d); } // kernels.cpp:24
__device__ __forceinline__ double dmin(double a, double b) { return (b < a) ? b : a; } // std::min
__device__ __forceinline__ double dmax(double a, double b) { return (a < b) ? b : a; } // std::max

// r2 > thr(h) guarantees fl(fl(sqrt(r2)) * inv_h) >= 2.5, i.e. the reference would return
// at its support test; skipping such pairs before the sqrt changes no bit of the result.
__device__ __forceinline__ double support_threshold(double inv_h) {
  double R = 2.5 / inv_h;
  return R * R * (1.0 + 1.0e-9);
}

} // namespace

__device__ __forceinline__ int hi_word(double v) { return __double2hiint(v); }

struct ExactPolicy {
  static constexpr bool kExactOrder = true;
  struct DI { double x, y, vx, vy, inv_h, thr; };
  struct DA { double rho, wcount, rho_dh, rot_v, div_v; };
  struct MW { double wc; double inv_h; };

  __device__ static DI den_i(double x, double y, double vx, double vy, double h) {
    DI I;
    I.x = x; I.y = y; I.vx = vx; I.vy = vy;
    I.inv_h = 1.0 / h;
    I.thr = support_threshold(I.inv_h);
    return I;
  }
  __device__ static DA den_zero() { return DA{0.0, 0.0, 0.0, 0.0, 0.0}; }
  __device__ static MW mw_zero() { return MW{kernel_w(0.0), 0.0}; }
  __device__ static double mw_value(const MW &m) { return m.wc; }

  // density_pair<kMask=false>, kernels.cpp:97-119
  template <bool MINIMG>
  __device__ static void den_pair(const DI &I, double2 xj, double2 vj, double mj, DA &s) {
    double dx0 = min_image(I.x - xj.x);
    double dx1 = min_image(I.y - xj.y);
    double r2 = dx0 * dx0 + dx1 * dx1;
    if (r2 <= 0.0) return;
    if (r2 > I.thr) return;
    double r = sqrt(r2);
    double q = r * I.inv_h;
    if (!(q < kSupport)) return;
    double w = kernel_w(q);
    double dw = kernel_dw(q);
    s.rho += mj * w;
    s.wcount += w;
    s.rho_dh -= mj * (2.0 * w + q * dw);
    double dv0 = I.vx - vj.x;
    double dv1 = I.vy - vj.y;
    double fac = mj * dw / r;
    s.div_v -= fac * (dv0 * dx0 + dv1 * dx1);
    s.rot_v += fac * (dv0 * dx1 - dv1 * dx0);
  }

  template <bool MINIMG>
  __device__ static void den_tile(const DI &I, const DenTile &T, DA &s) {
#pragma unroll 2
    for (int j = 0; j < kTJ; ++j) den_pair<MINIMG>(I, T.xy[j], T.vv[j], T.m[j], s);
  }

  template <bool MINIMG>
  __device__ static void mw_tile(const DI &I, const DenTile &T, MW &m) {
#pragma unroll 2
    for (int j = 0; j < kTJ; ++j) mw_pair<MINIMG>(I, T.xy[j], m);
  }

  // mean_wcount inner loop, grid.cpp:39-48
  template <bool MINIMG>
  __device__ static void mw_pair(const DI &I, double2 xj, MW &m) {
    double dx0 = I.x - xj.x;
    double dx1 = I.y - xj.y;
    dx0 -= round(dx0);
    dx1 -= round(dx1);
    double r2 = dx0 * dx0 + dx1 * dx1;
    if (r2 <= 0.0) return;
    if (r2 > I.thr) return;
    double q = sqrt(r2) * I.inv_h;
    if (q < kSupport) m.wc += kernel_w(q);
  }

  // density_step, kernels.cpp:184-192. 0 = Again (h updated), 1 = Done, 2 = Fail.
  __device__ static int den_step(const DA &s, double &h, double target, double h_max, int iter) {
    double wc = s.wcount + kernel_w(0.0);
    double ratio = sqrt(target / wc);
    if (fabs(ratio - 1.0) < 1.0e-4) return 1;
    double hn = dmin(h_max, h * dmin(1.2, dmax(0.8, ratio)));
    if (hn == h) return 1;
    if (iter >= 29) return 2;
    h = hn;
    return 0;
  }

  // density_publish, kernels.cpp:194-202
  __device__ static void den_publish(const DA &s, double h, double mi, double o[6]) {
    double w0 = kernel_w(0.0);
    double inv_h = 1.0 / h;
    double inv_h2 = inv_h * inv_h;
    double inv_h3 = inv_h2 * inv_h;
    o[0] = h;
    o[1] = (s.rho + mi * w0) * inv_h2;
    o[2] = s.wcount + w0;
    o[3] = (s.rho_dh - 2.0 * mi * w0) * inv_h3;
    o[4] = s.rot_v * inv_h3;
    o[5] = s.div_v * inv_h3;
  }

  struct FCold { double pad; };
  struct FI { double x0, x1, v0, v1, hi, inv_hi, inv_hi3, pri, bi, eps2, ci, thr; };
  struct FA { double a0, a1, udt, vsig, hdt; };

  // force_inv, kernels.cpp:155-172
  __device__ static FI for_i(double2 x, double2 vp, double h, double p, double rho,
                             double rho_dh, double c, double div_v, double rot_v, double,
                             FCold *) {
    FI I;
    I.x0 = x.x; I.x1 = x.y; I.v0 = vp.x; I.v1 = vp.y;
    I.hi = h;
    I.inv_hi = 1.0 / I.hi;
    I.inv_hi3 = I.inv_hi * I.inv_hi * I.inv_hi;
    double rhoi = rho;
    I.pri = p / (rhoi * rhoi) * (1.0 + 0.5 * I.hi * rho_dh / rhoi);
    double adiv = fabs(div_v);
    I.ci = c;
    I.bi = adiv / (adiv + fabs(rot_v) + 0.0001 * I.ci * I.inv_hi);
    I.eps2 = 0.01 * I.hi * I.hi;
    I.thr = support_threshold(I.inv_hi);
    return I;
  }
  __device__ static FA for_zero(double h_dt) { return FA{0.0, 0.0, 0.0, 0.0, h_dt}; }

  // Per-j terms hoisted into the tile with the reference's own operations:
  // grav*mj (kernels.cpp:129), pj/(rhoj*rhoj) (:142), mj/rhoj (:152).
  __device__ static double4 stage_force(double m, double rho, double p, double grav) {
    return make_double4(m, grav * m, p / (rho * rho), m / rho);
  }

  // force_pair<kMask=false>, kernels.cpp:121-153
  template <bool MINIMG>
  __device__ static void for_pair(const FI &I, double2 xj, double2 vj, double2 mg, double2 pv,
                                  double cj, FA &s) {
    double dx0 = min_image(I.x0 - xj.x);
    double dx1 = min_image(I.x1 - xj.y);
    double r2 = dx0 * dx0 + dx1 * dx1;
    if (r2 <= 0.0) return;
    double mj = mg.x;
    double soft = r2 + I.eps2;
    double gfac = mg.y / (soft * sqrt(soft));
    s.a0 -= gfac * dx0;
    s.a1 -= gfac * dx1;
    if (r2 > I.thr) return;
    double r = sqrt(r2);
    double q = r * I.inv_hi;
    if (!(q < kSupport)) return;
    double dwi = kernel_dw(q) * I.inv_hi3;
    double inv_r = 1.0 / r;
    double prj = pv.x;
    double acc = mj * (I.pri + prj) * dwi * inv_r;
    s.a0 -= acc * dx0;
    s.a1 -= acc * dx1;
    double dv0 = I.v0 - vj.x;
    double dv1 = I.v1 - vj.y;
    double dvdr = dv0 * dx0 + dv1 * dx1;
    s.udt += mj * I.pri * dwi * dvdr * inv_r;
    double mu = dmin(0.0, dvdr * inv_r);
    s.vsig = dmax(s.vsig, 1.0 * (I.ci + cj - 3.0 * mu * I.bi));
    s.hdt -= pv.y * dvdr * inv_r * dwi * 0.5 * I.hi;
  }

  __device__ static void for_tile_far(const FI &I, const ForTile &T, FA &s) {
    for_tile<true>(I, T, s); // never used: EXACT walks every chunk as near
  }

  template <bool MINIMG>
  __device__ static void for_tile(const FI &I, const ForTile &T, FA &s) {
#pragma unroll 2
    for (int j = 0; j < kTJ; ++j) for_pair<MINIMG>(I, T.xy[j], T.vv[j], T.mg[j], T.pv[j], T.c[j], s);
  }

  __device__ static void for_publish(const FI &, const FA &s, double o[5]) {
    o[0] = s.a0; o[1] = s.a1; o[2] = s.udt; o[3] = s.vsig; o[4] = s.hdt;
  }
};

// ---------------------------------------------------------------------------------------
// Streaming kernels: drift / kick1 / kick2 (kernels.cpp:305-341), one thread per slot.
// ---------------------------------------------------------------------------------------
template <bool AOS>
__global__ void __launch_bounds__(256) drift_kernel(Particle *aos, SoaMirror f, int n, double dt) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  if constexpr (AOS) {
    Particle &p = aos[s];
    double2 x = *reinterpret_cast<double2 *>(p.x);
    const double2 vp = *reinterpret_cast<const double2 *>(p.v_pred);
    const int32_t frozen = p.frozen;
    const double u = p.u, u_dt = p.u_dt;
    double adv = frozen ? 0.0 : dt;
    x.x += adv * vp.x;
    x.y += adv * vp.y;
    *reinterpret_cast<double2 *>(p.x) = x;
    p.u_pred = u + 0.5 * adv * u_dt;
    p.moved = frozen ? 0 : 1;
  } else {
    double2 x = f.x[s];
    const double2 vp = f.vp[s];
    const int32_t frozen = f.frozen[s];
    double adv = frozen ? 0.0 : dt;
    x.x += adv * vp.x;
    x.y += adv * vp.y;
    f.x[s] = x;
    f.u_pred[s] = f.u[s] + 0.5 * adv * f.u_dt[s];
    f.moved[s] = frozen ? 0 : 1;
  }
}

template <bool AOS>
__global__ void __launch_bounds__(256) kick1_kernel(Particle *aos, SoaMirror f, int n, double dt) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  double2 v, a;
  double u, u_dt;
  if constexpr (AOS) {
    const Particle &p = aos[s];
    v = *reinterpret_cast<const double2 *>(p.v);
    a = *reinterpret_cast<const double2 *>(p.a);
    u = p.u;
    u_dt = p.u_dt;
  } else {
    v = f.v[s];
    a = f.a[s];
    u = f.u[s];
    u_dt = f.u_dt[s];
  }
  double half = 0.5 * dt;
  v.x += half * a.x;
  v.y += half * a.y;
  u += half * u_dt;
  double vn = sqrt(v.x * v.x + v.y * v.y);
  double an = sqrt(a.x * a.x + a.y * a.y);
  double dtn = dmin(0.005 / (vn + 1.0e-12), sqrt(0.005 / (an + 1.0e-12)));
  if constexpr (AOS) {
    Particle &p = aos[s];
    *reinterpret_cast<double2 *>(p.v) = v;
    p.u = u;
    p.dt_next = dtn;
  } else {
    f.v[s] = v;
    f.u[s] = u;
    f.dt_next[s] = dtn;
  }
}

template <bool AOS>
__global__ void __launch_bounds__(256) kick2_kernel(Particle *aos, SoaMirror f, int n, double dt,
                                                    double gamma, double cfl) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  double2 v, a;
  double dbg0, u, u_dt, u_pred, rho, dt_next, h, v_sig;
  if constexpr (AOS) {
    const Particle &p = aos[s];
    v = *reinterpret_cast<const double2 *>(p.v);
    a = *reinterpret_cast<const double2 *>(p.a);
    dbg0 = p.dbg[0]; u = p.u; u_dt = p.u_dt; u_pred = p.u_pred; rho = p.rho;
    dt_next = p.dt_next; h = p.h; v_sig = p.v_sig;
  } else {
    v = f.v[s]; a = f.a[s]; dbg0 = f.dbg0[s]; u = f.u[s]; u_dt = f.u_dt[s];
    u_pred = f.u_pred[s]; rho = f.rho[s]; dt_next = f.dt_next[s]; h = f.h[s]; v_sig = f.v_sig[s];
  }
  double half = 0.5 * dt;
  v.x += half * a.x;
  v.y += half * a.y;
  u += half * (u_dt + dbg0);
  if (u < 0.5 * u_pred) u = 0.5 * u_pred;
  u_pred = u;
  double c = sqrt(gamma * (gamma - 1.0) * dmax(u, 1.0e-12));
  double pr = (gamma - 1.0) * rho * u;
  dt_next = dmin(dt_next, cfl * h / dmax(v_sig, c + c));
  if constexpr (AOS) {
    Particle &p = aos[s];
    *reinterpret_cast<double2 *>(p.v) = v;
    *reinterpret_cast<double2 *>(p.v_pred) = v;
    p.u = u; p.u_pred = u_pred; p.c = c; p.p = pr; p.dt_next = dt_next; p.h_dt = 0.0;
  } else {
    f.v[s] = v; f.vp[s] = v; f.u[s] = u; f.u_pred[s] = u_pred; f.c[s] = c; f.p[s] = pr;
    f.dt_next[s] = dt_next; f.h_dt[s] = 0.0;
  }
}

// EOS refresh of make_particles (grid.cpp:137-140), AoS mirror.
__global__ void eos_kernel(Particle *aos, int n, double gamma) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  Particle &p = aos[s];
  p.p = (gamma - 1.0) * p.rho * p.u;
  p.c = sqrt(gamma * (gamma - 1.0) * p.u);
}

// ---------------------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------------------
void launch_density_exact(const DenArgs &a, int n_items, bool aos, bool meanw, cudaStream_t s) {
  if (n_items <= 0) return;
  DenArgs b = a;
  b.n_items = n_items;
  const int G = pair_grid(n_items), B = kWarpsPerCta * 32;
  if (aos) {
    if (meanw) density_round_kernel<ExactPolicy, true, true><<<G, B, 0, s>>>(b);
    else density_round_kernel<ExactPolicy, true, false><<<G, B, 0, s>>>(b);
  } else {
    if (meanw) density_round_kernel<ExactPolicy, false, true><<<G, B, 0, s>>>(b);
    else density_round_kernel<ExactPolicy, false, false><<<G, B, 0, s>>>(b);
  }
}

void launch_force_exact(const ForArgs &a, int n_items, bool aos, cudaStream_t s) {
  if (n_items <= 0) return;
  ForArgs b = a;
  b.n_items = n_items;
  const int G = pair_grid(n_items), B = kWarpsPerCta * 32;
  if (aos) force_kernel<ExactPolicy, true, false><<<G, B, 0, s>>>(b);
  else force_kernel<ExactPolicy, false, false><<<G, B, 0, s>>>(b);
}

void launch_linear(int kernel, bool aos, Particle *p, const SoaMirror &f, int n, const Params &par,
                   cudaStream_t s) {
  if (n <= 0) return;
  const int B = 256, G = (n + B - 1) / B;
  if (kernel == 2) {
    if (aos) drift_kernel<true><<<G, B, 0, s>>>(p, f, n, par.dt);
    else drift_kernel<false><<<G, B, 0, s>>>(p, f, n, par.dt);
  } else if (kernel == 3) {
    if (aos) kick1_kernel<true><<<G, B, 0, s>>>(p, f, n, par.dt);
    else kick1_kernel<false><<<G, B, 0, s>>>(p, f, n, par.dt);
  } else {
    if (aos) kick2_kernel<true><<<G, B, 0, s>>>(p, f, n, par.dt, par.gamma, par.cfl);
    else kick2_kernel<false><<<G, B, 0, s>>>(p, f, n, par.dt, par.gamma, par.cfl);
  }
}

void launch_eos(Particle *p, int n, double gamma, cudaStream_t s) {
  if (n <= 0) return;
  eos_kernel<<<(n + 255) / 256, 256, 0, s>>>(p, n, gamma);
}

// Exact support fractions of the current state ("count f_* exactly per run,
// device counters in a validation pass"): over every active pair (i, j) of every local i,
// q = sqrt(r2) * (1/h_i) by the reference's arithmetic (kernels.cpp:24, :100-105: minimum
// image, r2 without contraction, IEEE sqrt and division; this file is built with
// --fmad=false) and counts of q < 2.5, < 1.5, < 0.5 (r2 > 0). One warp per work item, lane =
// local, every lane reading the same j (broadcast). Not on the timed path.
__global__ void __launch_bounds__(128) pair_fraction_kernel(Geom g, const Item *items, int n_items,
                                                            const int *list, SoaMirror f,
                                                            unsigned long long *cnt) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= n_items) return;
  const Item it = items[w];
  const bool live = lane < it.count;
  const int slot = list[it.start + (live ? lane : 0)];
  const double2 xi = f.x[slot];
  const double inv_h = 1.0 / f.h[slot];
  const Stencil st = make_stencil(it.cell, g.nx, g.ny);
  unsigned c25 = 0, c15 = 0, c05 = 0;
  for (int k = 0; k < st.n; ++k) {
    const int b = g.cell_begin[st.cell[k]], e = g.cell_begin[st.cell[k] + 1];
    for (int sj = b; sj < e; ++sj) {
      const double2 xj = f.x[sj];
      const double d0 = min_image(xi.x - xj.x), d1 = min_image(xi.y - xj.y);
      const double r2 = d0 * d0 + d1 * d1;
      if (!(r2 > 0.0)) continue;
      const double q = sqrt(r2) * inv_h;
      c25 += q < 2.5;
      c15 += q < 1.5;
      c05 += q < 0.5;
    }
  }
  if (!live) c25 = c15 = c05 = 0;
  for (int o = 16; o > 0; o >>= 1) {
    c25 += __shfl_xor_sync(0xffffffffu, c25, o);
    c15 += __shfl_xor_sync(0xffffffffu, c15, o);
    c05 += __shfl_xor_sync(0xffffffffu, c05, o);
  }
  if (lane == 0) {
    atomicAdd(cnt + 0, (unsigned long long)c25);
    atomicAdd(cnt + 1, (unsigned long long)c15);
    atomicAdd(cnt + 2, (unsigned long long)c05);
  }
}

void launch_pair_fractions(const Geom &g, const Item *items, int n_items, const int *list,
                           const SoaMirror &f, unsigned long long *cnt, cudaStream_t s) {
  cudaMemsetAsync(cnt, 0, 3 * sizeof(unsigned long long), s);
  if (n_items <= 0) return;
  pair_fraction_kernel<<<(n_items + 3) / 4, 128, 0, s>>>(g, items, n_items, list, f, cnt);
}

} // namespace sphb
