// kernels_fast.cu — FAST numerics for the two pair sweeps.
//
// Same skeleton as EXACT (pair_kernels.cuh); the per-pair arithmetic is restructured for
// the B200 FP64 pipe (64 DFMA/clk/SM) while staying a full-precision FP64 evaluation:
//   * periodic images are resolved once per stencil cell (shift folded into the staged j
//     position) instead of d - round(d) per pair (needs nx, ny >= 5, else min image);
//   * the support test compares the high 32 bits of r^2 and (2.5 h)^2 as integers (ALU
//     pipe, not FP64 pipe); pairs within 2^-20 of the support edge, where W ~ 1e-23, are
//     treated as outside. Out-of-support density pairs cost 2 DADD + DMUL + DFMA;
//   * sqrt and '/' become rsqrt.approx.f64 (MUFU) + a 2nd-order series correction (~1 ulp);
//   * the M5 spline is a Horner polynomial in s = 1.5 - q or 2.5 - q with selected
//     coefficients (no cancellation), plus a rarely-taken correction for q < 0.5;
//     dW/dq = -4 N E(s); the normalisation N, the -4 and the per-i constants (1/h^3,
//     P_i/rho_i^2 ...) are applied once per particle, not per pair;
//   * per-j invariants grav*m, m*p/rho^2, m/rho are hoisted into the shared-memory tile;
//   * each tile is consumed two pairs at a time with independent dependency chains.
// Summation order per particle is still the reference's j order; differences come from
// FMA contraction and the reassociated constant factors (~1e-15 relative per term).
#include "pair_kernels.cuh"
#include "sph_kernels.h"

namespace sphb {

namespace {

// x^(-1/2) and x^(-3/2) to ~1 ulp from the MUFU seed y0 = rsqrt.approx.f64(x), whose
// relative error is below 2^-20 (measured on B200, tools/rsq_probe). With e = 1 - x y0^2
// (|e| < 2^-19; y0 has 21 significant bits so y0^2 is exact and e is rounded once):
//   x^(-1/2) = y0 (1 + e/2 + 3e^2/8 + O(e^3)),   x^(-3/2) = y0^3 (1 + 3e/2 + 15e^2/8 + O(e^3)),
// truncation < 2^-55. 5 (resp. 6) FP64 ops instead of Newton's 7 (resp. 9).
__device__ __forceinline__ double rsqrt_seed(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
__device__ __forceinline__ double rsqrt_fast(double x) {
  const double y0 = rsqrt_seed(x);
  const double e = fma(-x, y0 * y0, 1.0);
  return fma(y0, e * fma(e, 0.375, 0.5), y0);
}
__device__ __forceinline__ double rsqrt3_fast(double x) {
  const double y0 = rsqrt_seed(x);
  const double t = y0 * y0;
  const double e = fma(-x, t, 1.0);
  const double y3 = t * y0;
  return fma(y3, e * fma(e, 1.875, 1.5), y3);
}

__device__ __forceinline__ int hi_word(double v) { return __double2hiint(v); }
// 0 < r2 < H2 as one unsigned compare on the high words (r2 >= 0 always): excludes the
// self pair (r2 == 0) and everything at or beyond the support edge, on the ALU pipe.
__device__ __forceinline__ bool in_support(double r2, unsigned hiH2m1) {
  return (unsigned)hi_word(r2) - 1u < hiH2m1;
}

// M5 spline (spline.hpp:12-41) as W(q) = N P(s), dW/dq = -4 N E(s):
//   q in [1.5, 2.5): s = 2.5 - q, P = s^4,                          E = s^3
//   q in [0.5, 1.5): s = 1.5 - q, P = -4s^4 + 4s^3 + 6s^2 + 4s + 1, E = -4s^3 + 3s^2 + 3s + 1
//   q in [0.0, 0.5): s = q,       P = 6s^4 - 15s^2 + 14.375,        E = -6s^3 + 7.5s
// (SPH_SPLINE3: one Horner with three-way selected coefficients; otherwise the innermost
// piece is the middle one plus the correction 10 t^4 / 10 t^3, t = 0.5 - q).
// The two outer pieces share Horner evaluation with selected coefficients (c4 == e3,
// c3 == c1, c0 == e0, e2 == e1), the innermost correction is a rarely-divergent branch.
struct Spline {
  double P, E;
  template <bool NEED_P>
  __device__ __forceinline__ void eval(double q) {
    // interval tests on the high word: for q >= 0, q < 1.5 <=> hi(q) < hi(1.5) exactly
    // (1.5 and 0.5 have zero low words), so they run on the ALU pipe
    const int hq = hi_word(q);
    const bool mid = hq < 0x3FF80000;  // q < 1.5
#if SPH_SPLINE3
    // three-way coefficient select, local variable s = 2.5 - q | 1.5 - q | q
    const bool inner = hq < 0x3FE00000; // q < 0.5
    const double s = inner ? q : (mid ? 1.5 : 2.5) - q;
    const double e3 = inner ? -6.0 : (mid ? -4.0 : 1.0), e2 = (mid && !inner) ? 3.0 : 0.0;
    const double e1 = inner ? 7.5 : (mid ? 3.0 : 0.0), e0 = (mid && !inner) ? 1.0 : 0.0;
    E = fma(fma(fma(e3, s, e2), s, e1), s, e0);
    if (NEED_P) {
      const double c4 = inner ? 6.0 : (mid ? -4.0 : 1.0), c31 = (mid && !inner) ? 4.0 : 0.0;
      const double c2 = inner ? -15.0 : (mid ? 6.0 : 0.0), c0 = inner ? 14.375 : (mid ? 1.0 : 0.0);
      P = fma(fma(fma(fma(c4, s, c31), s, c2), s, c31), s, c0);
    }
#else
    const double s = (mid ? 1.5 : 2.5) - q;
    const double c4 = mid ? -4.0 : 1.0, c31 = mid ? 4.0 : 0.0, c2 = mid ? 6.0 : 0.0;
    const double c0 = mid ? 1.0 : 0.0, e21 = mid ? 3.0 : 0.0;
    E = fma(fma(fma(c4, s, e21), s, e21), s, c0);
    if (NEED_P) P = fma(fma(fma(fma(c4, s, c31), s, c2), s, c31), s, c0);
    if (__builtin_expect(hq < 0x3FE00000, 0)) { // q < 0.5: ~4 % of in-support pairs
      const double t = 0.5 - q, t2 = t * t, t3 = t2 * t;
      E = fma(10.0, t3, E);
      if (NEED_P) P = fma(10.0, t3 * t, P);
    }
#endif
  }
};

} // namespace

struct FastPolicy {
  static constexpr bool kExactOrder = false;
  static constexpr double kW0 = kNorm2d * 14.375; // kernel_w(0)

  struct DI { double x, y, vx, vy, inv_h; unsigned hiH2m1; };
  // Scaled sums (N = spline normalisation): rho = N*S_rho, wcount = N*S_w,
  // rho_dh = -N*(2 S_rho - 4 S_qE), div_v = 4N*S_div, rot_v = -4N*S_rot (all / h^2, h^3).
  struct DA { double rho, w, qe, rot, div; };
  struct MW { double w; };

  __device__ static DI den_i(double x, double y, double vx, double vy, double h) {
    DI I;
    I.x = x; I.y = y; I.vx = vx; I.vy = vy;
    I.inv_h = 1.0 / h;
    I.hiH2m1 = (unsigned)hi_word(6.25 * h * h) - 1u;
    return I;
  }
  __device__ static DA den_zero() { return DA{0.0, 0.0, 0.0, 0.0, 0.0}; }
  __device__ static MW mw_zero() { return MW{0.0}; }
  __device__ static double mw_value(const MW &m) { return kW0 + kNorm2d * m.w; }

  __device__ __forceinline__ static void den_in(const DI &I, double dx, double dy, double r2,
                                                double2 vj, double mj, DA &s) {
    const double rinv = rsqrt_fast(r2);
    const double q = r2 * rinv * I.inv_h;
    Spline sp;
    sp.template eval<true>(q);
    s.rho = fma(mj, sp.P, s.rho);
    s.w += sp.P;
    const double mE = mj * sp.E;
    s.qe = fma(q, mE, s.qe);
    const double fac = mE * rinv;
    const double dvx = I.vx - vj.x, dvy = I.vy - vj.y;
    s.div = fma(fac, fma(dvx, dx, dvy * dy), s.div);
    s.rot = fma(fac, fma(dvx, dy, -dvy * dx), s.rot);
  }

  // Four pairs per step: the four distance chains are straight-line code (independent,
  // interleaved by the scheduler), then the in-support blocks run in j order.
  template <bool MINIMG>
  __device__ static void den_tile(const DI &I, const DenTile &T, DA &s) {
#pragma unroll 2
    for (int j = 0; j < kTJ; j += 4) {
      double dx[4], dy[4], r2[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double2 xj = T.xy[j + k];
        dx[k] = I.x - xj.x;
        dy[k] = I.y - xj.y;
        if (MINIMG) { dx[k] -= round(dx[k]); dy[k] -= round(dy[k]); }
        r2[k] = fma(dx[k], dx[k], dy[k] * dy[k]);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (in_support(r2[k], I.hiH2m1)) den_in(I, dx[k], dy[k], r2[k], T.vv[j + k], T.m[j + k], s);
    }
  }

  template <bool MINIMG>
  __device__ static void mw_tile(const DI &I, const DenTile &T, MW &m) {
#pragma unroll 4
    for (int j = 0; j < kTJ; ++j) {
      double dx = I.x - T.xy[j].x, dy = I.y - T.xy[j].y;
      if (MINIMG) { dx -= round(dx); dy -= round(dy); }
      const double r2 = fma(dx, dx, dy * dy);
      if (in_support(r2, I.hiH2m1)) {
        Spline sp;
        sp.template eval<true>(r2 * rsqrt_fast(r2) * I.inv_h);
        m.w += sp.P;
      }
    }
  }

  // density_step (kernels.cpp:184-192) on the scaled sums.
  __device__ static int den_step(const DA &s, double &h, double target, double h_max, int iter) {
    const double wc = fma(kNorm2d, s.w, kW0);
    const double ratio = sqrt(target / wc);
    if (fabs(ratio - 1.0) < 1.0e-4) return 1;
    const double f = fmin(1.2, fmax(0.8, ratio));
    const double hn = fmin(h_max, h * f);
    if (hn == h) return 1;
    if (iter >= 29) return 2;
    h = hn;
    return 0;
  }

  // density_publish (kernels.cpp:194-202).
  __device__ static void den_publish(const DA &s, double h, double mi, double o[6]) {
    const double inv_h = 1.0 / h;
    const double inv_h2 = inv_h * inv_h;
    const double inv_h3 = inv_h2 * inv_h;
    const double n3 = kNorm2d * inv_h3;
    o[0] = h;
    o[1] = fma(kNorm2d, s.rho, mi * kW0) * inv_h2;
    o[2] = fma(kNorm2d, s.w, kW0);
    // reference: rho_dh = (sum -m(2w + q dw) - 2 m_i w0) / h^3, dw = -4 N E
    o[3] = -fma(kNorm2d, fma(-4.0, s.qe, 2.0 * s.rho), 2.0 * mi * kW0) * inv_h3;
    o[4] = -4.0 * s.rot * n3;
    o[5] = 4.0 * s.div * n3;
  }

#if SPH_COLD
  // per-i constants used only on the in-support path and at publish live in shared memory
  // (one slot per lane), keeping the hot loop's register footprint small
  struct FCold { double vx, vy, pri, mb3, K, ci, hi, pad; };
  struct FI { double x, y, inv_hi, eps2; unsigned hiH2m1; FCold *cold; };
#else
  struct FCold { double pad; };
  struct FI { double x, y, vx, vy, inv_hi, eps2, pri, mb3, ci, hi, K; unsigned hiH2m1; };
#endif

  struct FA { double ax, ay, udt, vsig, hdt, hdt0; };

  // force_inv (kernels.cpp:155-172); K = -4 N / h^3 multiplies every SPH pair term.
  __device__ static FI for_i(double2 x, double2 vp, double h, double p, double rho,
                             double rho_dh, double c, double div_v, double rot_v, double,
                             FCold *cold) {
    FI I;
    I.x = x.x; I.y = x.y;
    I.inv_hi = 1.0 / h;
    I.hiH2m1 = (unsigned)hi_word(6.25 * h * h) - 1u;
    I.eps2 = 0.01 * h * h;
    const double irho = 1.0 / rho;
    const double pri = p * irho * irho * fma(0.5 * h * rho_dh, irho, 1.0);
    const double adiv = fabs(div_v);
    const double bi = adiv / (adiv + fabs(rot_v) + 0.0001 * c * I.inv_hi);
    const double K = -4.0 * kNorm2d * I.inv_hi * I.inv_hi * I.inv_hi;
#if SPH_COLD
    cold->vx = vp.x; cold->vy = vp.y; cold->pri = pri; cold->mb3 = -3.0 * bi; cold->K = K;
    cold->ci = c; cold->hi = h;
    I.cold = cold;
#else
    (void)cold;
    I.vx = vp.x; I.vy = vp.y; I.pri = pri; I.mb3 = -3.0 * bi; I.K = K; I.ci = c; I.hi = h;
#endif
    return I;
  }
  __device__ static FA for_zero(double h_dt) { return FA{0.0, 0.0, 0.0, -1.0, 0.0, h_dt}; }

  // tile terms: (m, grav*m, m*p/rho^2, m/rho)
  __device__ static double4 stage_force(double m, double rho, double p, double grav) {
    const double irho = 1.0 / rho;
    const double V = m * irho;
    return make_double4(m, grav * m, V * p * irho, V);
  }

  // SPH part of force_pair for one in-support pair; returns the radial factor to add to
  // the gravity factor (both multiply dx, dy).
  __device__ __forceinline__ static double for_in(const FI &I, double dx, double dy, double r2,
                                                  double2 vj, double2 mg, double2 pv, double cj,
                                                  FA &s) {
#if SPH_COLD
    const FCold &C = *I.cold;
#else
    const FI &C = I;
#endif
    const double rinv = rsqrt_fast(r2);
    const double q = r2 * rinv * I.inv_hi;
    Spline sp;
    sp.template eval<false>(q);
    const double g = sp.E * rinv;
    const double dvx = C.vx - vj.x, dvy = C.vy - vj.y;
    const double dvdr = fma(dvx, dx, dvy * dy);
    const double gd = g * dvdr;
    s.udt = fma(mg.x, gd, s.udt);
    s.hdt = fma(pv.y, gd, s.hdt);
    // mu = min(0, dvdr / r): sign test on the high word (ALU), then one DMUL
    const double mu = (hi_word(dvdr) < 0 ? dvdr : 0.0) * rinv;
    // vsig = max_j (c_i + c_j - 3 mu b_i) = c_i + max_j (c_j - 3 mu b_i): fl(c_i + x) is
    // monotonic in x, so adding c_i once at the end gives the same value
    const double vs = fma(mu, C.mb3, cj);
    // both >= 0 (or the -1 sentinel, whose bit pattern is negative): signed 64-bit integer
    // order equals double order here, so the max runs on the ALU pipe
    if (__double_as_longlong(vs) > __double_as_longlong(s.vsig)) s.vsig = vs;
    return fma(mg.x, C.pri, pv.x) * g * C.K;
  }

  // Four pairs per step: distances and the softened gravity (every active pair,
  // kernels.cpp:128-131) are straight-line code for the four pairs, so their rsqrt /
  // Newton chains interleave; the divergent SPH blocks follow in j order. The self pair
  // has dx = dy = 0 and padding has gm = 0: both contribute exactly zero.
  template <bool MINIMG>
  __device__ static void for_tile(const FI &I, const ForTile &T, FA &s) {
    constexpr int G = SPH_FJ; // pairs whose gravity chains are interleaved
#pragma unroll 1
    for (int j = 0; j < kTJ; j += G) {
      double dx[G], dy[G], r2[G], f[G];
      bool in[G];
#pragma unroll
      for (int k = 0; k < G; ++k) {
        const double2 xj = T.xy[j + k];
        dx[k] = I.x - xj.x;
        dy[k] = I.y - xj.y;
        if (MINIMG) { dx[k] -= round(dx[k]); dy[k] -= round(dy[k]); }
        r2[k] = fma(dx[k], dx[k], dy[k] * dy[k]);
        f[k] = T.mg[j + k].y * rsqrt3_fast(r2[k] + I.eps2);
        in[k] = in_support(r2[k], I.hiH2m1);
      }
#if SPH_MERGE
      // one block for the whole group, chains interleaved; pairs outside the support are
      // evaluated on a safe r2 and their contributions selected away
      bool any = false;
#pragma unroll
      for (int k = 0; k < G; ++k) any |= in[k];
      if (any) {
#pragma unroll
        for (int k = 0; k < G; ++k) {
          const double add = for_in_masked(I, dx[k], dy[k], in[k] ? r2[k] : 1.0, in[k], T.vv[j + k],
                                           T.mg[j + k], T.pv[j + k], T.c[j + k], s);
          f[k] += add;
        }
      }
#else
#pragma unroll
      for (int k = 0; k < G; ++k)
        if (in[k])
          f[k] += for_in(I, dx[k], dy[k], r2[k], T.vv[j + k], T.mg[j + k], T.pv[j + k], T.c[j + k], s);
#endif
#pragma unroll
      for (int k = 0; k < G; ++k) {
        s.ax = fma(-f[k], dx[k], s.ax);
        s.ay = fma(-f[k], dy[k], s.ay);
      }
    }
  }

  // for_in with the contributions of a pair outside the support selected to zero
  __device__ __forceinline__ static double for_in_masked(const FI &I, double dx, double dy,
                                                         double r2, bool in, double2 vj,
                                                         double2 mg, double2 pv, double cj,
                                                         FA &s) {
#if SPH_COLD
    const FCold &C = *I.cold;
#else
    const FI &C = I;
#endif
    const double rinv = rsqrt_fast(r2);
    const double q = r2 * rinv * I.inv_hi;
    Spline sp;
    sp.template eval<false>(q);
    const double g = in ? sp.E * rinv : 0.0;
    const double dvx = C.vx - vj.x, dvy = C.vy - vj.y;
    const double dvdr = fma(dvx, dx, dvy * dy);
    const double gd = g * dvdr;
    s.udt = fma(mg.x, gd, s.udt);
    s.hdt = fma(pv.y, gd, s.hdt);
    const double mu = (hi_word(dvdr) < 0 ? dvdr : 0.0) * rinv;
    const double vs = fma(mu, C.mb3, cj);
    if (in && vs > s.vsig) s.vsig = vs;
    return fma(mg.x, C.pri, pv.x) * g * C.K;
  }

  // Gravity only (chunk out of every lane's support): branch-free, shifted images.
  __device__ static void for_tile_far(const FI &I, const ForTile &T, FA &s) {
#pragma unroll 4
    for (int j = 0; j < kTJ; ++j) {
      const double2 xj = T.xy[j];
      const double dx = I.x - xj.x, dy = I.y - xj.y;
      const double f = T.mg[j].y * rsqrt3_fast(fma(dx, dx, fma(dy, dy, I.eps2)));
      s.ax = fma(-f, dx, s.ax);
      s.ay = fma(-f, dy, s.ay);
    }
  }

  __device__ static void for_publish(const FI &I, const FA &s, double o[5]) {
#if SPH_COLD
    const FCold &C = *I.cold;
#else
    const FI &C = I;
#endif
    o[0] = s.ax;
    o[1] = s.ay;
    o[2] = C.pri * C.K * s.udt;
    o[3] = s.vsig < 0.0 ? 0.0 : C.ci + s.vsig;
    o[4] = fma(-0.5 * C.hi * C.K, s.hdt, s.hdt0);
  }
};

// j-view builders: gather the sweep's j fields into ilist order (+ hoisted invariants).
template <bool AOS>
__global__ void jview_density_kernel(double2 *xy, double2 *vv, double *m, const int *ilist,
                                     const Particle *aos, SoaMirror f, int n) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  JSrc<AOS> src;
  if constexpr (AOS) src.p = aos; else src.f = f;
  const int sj = ilist[p];
  xy[p] = src.x(sj);
  vv[p] = src.vp(sj);
  m[p] = src.m(sj);
}

template <bool AOS>
__global__ void jview_force_kernel(double2 *xy, double2 *vv, double2 *mg, double2 *pv, double *c,
                                   const int *ilist, const Particle *aos, SoaMirror f, int n,
                                   double grav) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  JSrc<AOS> src;
  if constexpr (AOS) src.p = aos; else src.f = f;
  const int sj = ilist[p];
  xy[p] = src.x(sj);
  vv[p] = src.vp(sj);
  const double4 d = FastPolicy::stage_force(src.m(sj), src.rho(sj), src.pr(sj), grav);
  mg[p] = make_double2(d.x, d.y);
  pv[p] = make_double2(d.z, d.w);
  c[p] = src.c(sj);
}

void launch_jview_density(double2 *xy, double2 *vv, double *m, const int *ilist,
                          const Particle *aos, const SoaMirror &f, bool use_aos, int n,
                          cudaStream_t s) {
  if (n <= 0) return;
  if (use_aos) jview_density_kernel<true><<<(n + 255) / 256, 256, 0, s>>>(xy, vv, m, ilist, aos, f, n);
  else jview_density_kernel<false><<<(n + 255) / 256, 256, 0, s>>>(xy, vv, m, ilist, aos, f, n);
}

void launch_jview_force(double2 *xy, double2 *vv, double2 *mg, double2 *pv, double *c,
                        const int *ilist, const Particle *aos, const SoaMirror &f, bool use_aos,
                        int n, double grav, cudaStream_t s) {
  if (n <= 0) return;
  if (use_aos)
    jview_force_kernel<true><<<(n + 255) / 256, 256, 0, s>>>(xy, vv, mg, pv, c, ilist, aos, f, n, grav);
  else
    jview_force_kernel<false><<<(n + 255) / 256, 256, 0, s>>>(xy, vv, mg, pv, c, ilist, aos, f, n, grav);
}

void launch_density_fast(const DenArgs &a, int n_items, bool aos, cudaStream_t s) {
  if (n_items <= 0) return;
  DenArgs b = a;
  b.n_items = n_items;
  const int G = pair_grid(n_items), B = kWarpsPerCta * 32;
  if (b.boxes && b.jlist) {
    if (aos) density_cull_kernel<FastPolicy, true><<<G, B, 0, s>>>(b);
    else density_cull_kernel<FastPolicy, false><<<G, B, 0, s>>>(b);
  } else {
    if (aos) density_round_kernel<FastPolicy, true, false><<<G, B, 0, s>>>(b);
    else density_round_kernel<FastPolicy, false, false><<<G, B, 0, s>>>(b);
  }
}

void launch_force_fast(const ForArgs &a, int n_items, bool aos, cudaStream_t s) {
  if (n_items <= 0) return;
  ForArgs b = a;
  b.n_items = n_items;
  const int G = pair_grid(n_items), B = kWarpsPerCta * 32;
  if (b.jv.xy) {
    if (aos) force_kernel<FastPolicy, true, true><<<G, B, 0, s>>>(b);
    else force_kernel<FastPolicy, false, true><<<G, B, 0, s>>>(b);
  } else {
    if (aos) force_kernel<FastPolicy, true, false><<<G, B, 0, s>>>(b);
    else force_kernel<FastPolicy, false, false><<<G, B, 0, s>>>(b);
  }
}

} // namespace sphb
