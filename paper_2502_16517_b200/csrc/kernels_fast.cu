// kernels_fast.cu — FAST numerics for the two pair sweeps.
//
// Same skeleton as EXACT (pair_kernels.cuh); the per-pair arithmetic is restructured for
// the B200 FP64 pipe (64 DFMA/clk/SM) while staying a full-precision FP64 evaluation:
//   * periodic images are resolved once per stencil cell (shift folded into the staged j
//     position) instead of d - round(d) per pair (needs nx, ny >= 5, else min image);
//   * the support test compares the high 32 bits of r^2 and (2.5 h)^2 as integers (ALU
//     pipe, not FP64 pipe); density pairs within 2^-20 of the support edge, where W ~ 1e-23,
//     are treated as outside. Force pairs in that band are decided as the reference decides
//     them (support_cand / ref_support, bit for bit), because the v_sig max is not
//     continuous at the edge. Out-of-support density pairs cost 2 DADD + DMUL + DFMA;
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
// relative error is below 2^-20 (measured on B200, tools/fp64_micro.cu). With e = 1 - x y0^2
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

// Force pairs: the v_sig max (kernels.cpp:151) is discontinuous at the support edge (the
// other pair terms vanish there), so the edge is decided as the reference decides it.
// support_cand: 3 <= hi(r2) <= hi(H2) + 1 (r2 = 0 and denormal r2 excluded); support_sure:
// hi(r2) <= hi(H2) - 2, certainly q < 2.5 by any rounding. Candidates in between (a band of
// ~2^-19 relative width around (2.5 h)^2) take ref_support.
__device__ __forceinline__ bool support_cand(double r2, unsigned hiH2m1) {
  return (unsigned)hi_word(r2) - 3u < hiH2m1;
}
__device__ __forceinline__ bool support_sure(double r2, unsigned hiH2m1) {
  return (unsigned)hi_word(r2) < hiH2m1;
}
// IEEE sqrt (round to nearest) of a positive normal x without the library's special-case
// call: y ~ x^-1/2 to ~1 ulp, s = x y, then one residual step s + (x - s^2) y / 2 rounds
// correctly (tools/sqrt_probe.cu checks it against __dsqrt_rn).
__device__ __forceinline__ double sqrt_rn_normal(double x) {
  const double y = rsqrt_fast(x);
  const double s = __dmul_rn(x, y);
  const double r = __fma_rn(-s, s, x);
  return __fma_rn(r, 0.5 * y, s);
}
// kernels.cpp:124-136 bit for bit: r2 without contraction, IEEE sqrt, q = r * (1/h) < 2.5
// (r2 here is within 2^-18 of (2.5 h)^2: positive and normal)
__device__ __forceinline__ bool ref_support(double dx, double dy, double inv_h) {
  const double r2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
  return r2 > 0.0 && __dmul_rn(sqrt_rn_normal(r2), inv_h) < 2.5;
}
// ... from the unshifted positions, with the reference's minimum image (kernels.cpp:24)
__device__ __forceinline__ bool ref_support_xy(double xi0, double xi1, double xj0, double xj1,
                                            double inv_h) {
  double d0 = __dsub_rn(xi0, xj0), d1 = __dsub_rn(xi1, xj1);
  d0 = __dsub_rn(d0, round(d0));
  d1 = __dsub_rn(d1, round(d1));
  return ref_support(d0, d1, inv_h);
}

// M5 spline (spline.hpp:12-41) as W(q) = N P(s), dW/dq = -4 N E(s):
//   q in [1.5, 2.5): s = 2.5 - q, P = s^4,                          E = s^3
//   q in [0.5, 1.5): s = 1.5 - q, P = -4s^4 + 4s^3 + 6s^2 + 4s + 1, E = -4s^3 + 3s^2 + 3s + 1
//   q in [0.0, 0.5): s = q,       P = 6s^4 - 15s^2 + 14.375,        E = -6s^3 + 7.5s
// The innermost
// piece is the middle one plus the correction 10 t^4 / 10 t^3, t = 0.5 - q.
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

  struct FCold { double pad; };
  struct FI { double x, y, vx, vy, inv_hi, eps2, pri, mb3, ci, hi, K; unsigned hiH2m1; };

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
    (void)cold;
    I.vx = vp.x; I.vy = vp.y; I.pri = pri; I.mb3 = -3.0 * bi; I.K = K; I.ci = c; I.hi = h;
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
    const FI &C = I;
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
        // edge band: the reference's decision on this (dx, dy) (exact in the minimum-image
        // mode, where dx is the reference's; with the folded periodic shift dx may differ
        // from it in the last bit)
        in[k] = support_cand(r2[k], I.hiH2m1) &&
                (support_sure(r2[k], I.hiH2m1) || ref_support(dx[k], dy[k], I.inv_hi));
      }
#pragma unroll
      for (int k = 0; k < G; ++k)
        if (in[k])
          f[k] += for_in(I, dx[k], dy[k], r2[k], T.vv[j + k], T.mg[j + k], T.pv[j + k], T.c[j + k], s);
#pragma unroll
      for (int k = 0; k < G; ++k) {
        s.ax = fma(-f[k], dx[k], s.ax);
        s.ay = fma(-f[k], dy[k], s.ay);
      }
    }
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
    const FI &C = I;
    o[0] = s.ax;
    o[1] = s.ay;
    o[2] = C.pri * C.K * s.udt;
    o[3] = s.vsig < 0.0 ? 0.0 : C.ci + s.vsig;
    o[4] = fma(-0.5 * C.hi * C.K, s.hdt, s.hdt0);
  }
};

// ---------------------------------------------------------------------------------------
// Issue-lean FAST force sweep (force2). Same decomposition and numerics as force_kernel
// with the FAST policy (one warp per item, lane = local i, chunks of the spatially ordered
// active list, far chunks gravity-only), re-shaped so that the FP64 pipe, not instruction
// issue, is the limit. ncu on force_kernel showed ~44 issued instructions per pair of
// which only ~23 were FP64 (issue 63 %, FP64 pipe 65 %):
//   * chunks are staged with cp.async straight into a double-buffered per-warp tile (no
//     prefetch registers, no STS), the periodic image shift moves to the i side (xs, ys);
//   * the tile keeps the gravity fields as separate x[], y[], gm[] arrays so one LDS.128
//     serves two j's; the SPH fields are paired (vx,vy), (P,V), (c,m);
//   * the spline piece is picked from a 3-row coefficient table in shared memory
//     (E = Horner in q, kSplQ): no selects, no predicated correction for q < 0.5;
//   * the series constants come from the kernel parameters (constant-bank operands), so
//     they are not re-materialised with IMADs inside the loop.
// ---------------------------------------------------------------------------------------
struct __align__(16) F2Tile {
  double x[kTJ], y[kTJ], gm[kTJ];
  double2 vv[kTJ], pv[kTJ], cm[kTJ];
  double2 spl[9]; // spline coefficient table (kSplQ, 6 used), one copy per tile so rows
                  // are addressed relative to the tile pointer
  double vsig0[kTJ]; // each lane's v_sig before this chunk (force2_edge)
  int edge;          // nonzero: some lane met an edge-band pair in this chunk (force2_sph)
};


// spline.hpp:12-41 as dW/dq = -4 N E, E per piece (outer, mid, inner) as a polynomial in q:
// E = ((a3 q + a2) q + a1) q + a0, rows of two double2 {a3, a2}, {a1, a0}. (Round 1 used
// s = c_off - q; the q form saves that DFMA, which reads three registers: force -0.7 %.)
__constant__ double2 kSplQ[6] = {
    {-1.0, 7.5}, {-18.75, 15.625}, // (2.5 - q)^3
    {4.0, -15.0}, {15.0, -1.25},   // -4 s^3 + 3 s^2 + 3 s + 1, s = 1.5 - q
    {-6.0, 0.0}, {7.5, 0.0},       // 6 s^3 - 7.5 s, s = -q
};

__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// table row of q (q >= 0): 0 outer, 1 mid, 2 inner; interval tests on the high word
// (exact: 0.5 and 1.5 have zero low words)
__device__ __forceinline__ int spline_row(double q) {
  const int hq = __double2hiint(q);
  return (hq < 0x3FE00000 ? 1 : 0) + (hq < 0x3FF80000 ? 1 : 0);
}

// force2 / density2 CTA shape: W warps per CTA, MINB CTAs per SM requested from ptxas
// (registers <= 65536 / (32 W MINB)). Measured at 2^21 / ppc 1024 (ms, force / density
// round 0): 4 warps x 5 (96 regs) 33.31 / 19.07; 1 x 20 (96) 33.11 / 18.74; 1 x 16 (115)
// 33.48 / 19.68; 1 x 22 or 24 and 2 x 11 (80 regs, spills) 35.8-36.1 / 19.7-19.8.
#ifndef SPH_F2_WPC
#define SPH_F2_WPC 1
#endif
#ifndef SPH_MINB_F2
#define SPH_MINB_F2 20
#endif
#ifndef SPH_D2_WPC
#define SPH_D2_WPC 1
#endif
constexpr int kF2W = SPH_F2_WPC, kD2W = SPH_D2_WPC;
#ifndef SPH_F2_FARU
#define SPH_F2_FARU 2 // far loop unroll (groups of 4 pairs; 2: -0.4 %, 4: same as 2)
#endif
constexpr int kF2FarU = SPH_F2_FARU;
#ifndef SPH_F2_NEARU
#define SPH_F2_NEARU 8 // near loop unroll (pairs of pairs; r1: 2 -0.9 %, 4 -1.9 % vs 1; r2 with the
                       // persistent q-form kernel: 8 -0.7 % vs 4, 16 +19 %, profiles/r2u_unroll.txt)
#endif
constexpr int kF2NearU = SPH_F2_NEARU;
#ifndef SPH_D2_U
#define SPH_D2_U 1 // density round-0 pair loop unroll (groups of 4 pairs; 2: +1.5 %)
#endif
constexpr int kD2U = SPH_D2_U;
#ifndef SPH_D2_JU
#define SPH_D2_JU 4 // density j-slice (rounds >= 1) pair loop unroll (4: round 1 -1.4 %)
#endif
constexpr int kD2JU = SPH_D2_JU;

// SPH part of force_pair (kernels.cpp:132-152) for one in-support pair: accumulates u_dt,
// h_dt, v_sig and returns the SPH radial factor A*g (the caller applies K).
struct F2I { double vx, vy, inv_hi, pri, mb3; int hiQ05, hiQ15; };
// Candidates include the edge band (support_cand): there the u_dt, h_dt and acceleration
// terms are O(2^-57) whichever side of q = 2.5 the pair lies, but the v_sig max is not
// continuous. An edge pair flags the tile (a predicated shared store, no extra register:
// an extra live register makes ptxas rematerialise the tile address in every block, +5 %);
// force2_edge then redoes the flagged chunk's v_sig max from the value saved before it,
// taking edge pairs only where the reference would. The SPH block stays branch-free.
__device__ __forceinline__ double f2_rinv(double r2, double k0375) {
  const double y0 = rsqrt_seed(r2);
  const double e = fma(-r2, y0 * y0, 1.0);
  return fma(y0, e * fma(e, k0375, 0.5), y0);
}
__device__ __forceinline__ double force2_sph_r(const F2I &I, const F2Tile &T, int j, double dx,
                                               double dy, double r2, double rinv, double &udt,
                                               double &hdt, double &vsig, unsigned hiH2m1) {
  const int hr = __double2hiint(r2);
  int row = hr < I.hiQ15 ? 2 : 0;
  if (hr < I.hiQ05) row = 4;
  const double2 t1 = T.spl[row], t2 = T.spl[row + 1];
  const double q = (r2 * rinv) * I.inv_hi;
  const double E = fma(fma(fma(t1.x, q, t1.y), q, t2.x), q, t2.y);
  const double g = E * rinv;
  const double2 vj = T.vv[j];
  const double dvx = I.vx - vj.x, dvy = I.vy - vj.y;
  const double dvdr = fma(dvx, dx, dvy * dy);
  const double gd = g * dvdr;
  const double2 cm = T.cm[j], pv = T.pv[j];
  // gd in the same operand slot of both updates (reuse cache)
  udt = fma(gd, cm.y, udt);
  hdt = fma(gd, pv.y, hdt);
  const double mu = (__double2hiint(dvdr) < 0 ? dvdr : 0.0) * rinv;
  const double vs = fma(mu, I.mb3, cm.x);
  if (__double_as_longlong(vs) > __double_as_longlong(vsig)) vsig = vs;
  if ((unsigned)hr >= hiH2m1) const_cast<F2Tile &>(T).edge = hr;
  return fma(cm.y, I.pri, pv.x) * g;
}

__device__ __forceinline__ double force2_sph(const F2I &I, const F2Tile &T, int j, double dx,
                                             double dy, double r2, double k0375, double &udt,
                                             double &hdt, double &vsig, unsigned hiH2m1) {
  return force2_sph_r(I, T, j, dx, dy, r2, f2_rinv(r2, k0375), udt, hdt, vsig, hiH2m1);
}


// A flagged chunk's v_sig max redone from the value before it (kernels.cpp:124-151): the
// pairs certainly inside with force2_sph's arithmetic, the edge-band pairs only if the
// reference's support decision, from the unshifted positions, has them inside.
__device__ __forceinline__ double force2_edge(const F2I &I, const F2Tile &T, int lane, double2 xi,
                                              double xs, double ys, unsigned hiH2m1) {
  double vsig = T.vsig0[lane];
  for (int j = 0; j < kTJ; ++j) {
    const double dx = xs - T.x[j], dy = ys - T.y[j];
    const double r2 = fma(dx, dx, dy * dy);
    if (!support_cand(r2, hiH2m1)) continue;
    if (!support_sure(r2, hiH2m1) && !ref_support_xy(xi.x, xi.y, T.x[j], T.y[j], I.inv_hi))
      continue;
    const double rinv = rsqrt_fast(r2);
    const double2 vj = T.vv[j];
    const double dvdr = fma(I.vx - vj.x, dx, (I.vy - vj.y) * dy);
    const double vs = fma((__double2hiint(dvdr) < 0 ? dvdr : 0.0) * rinv, I.mb3, T.cm[j].x);
    if (__double_as_longlong(vs) > __double_as_longlong(vsig)) vsig = vs;
  }
  return vsig;
}

__device__ __forceinline__ void force2_stage(F2Tile &T, const ActiveLayout &L, const F2View &jv,
                                             int nb, int k, int lane) {
  const char *src = reinterpret_cast<const char *>(
      jv.blk + (size_t)chunk_box_index(L.base[nb], L.cell[nb], k) * kF2Blk);
  char *dst = reinterpret_cast<char *>(&T);
#pragma unroll
  for (int t = 0; t < 5; ++t) {
    const int piece = lane + 32 * t; // 144 pieces of 16 bytes
    if (piece < kF2Blk / 2) cp_async16(dst + 16 * piece, src + 16 * piece);
  }
  cp_async_commit();
}

// AOS layout (the layout ablation's AoS arm): the chunk's j fields come straight from the
// 272-B records, no j-view. Lane l copies j = 32 k + l of stencil cell nb: x, y, v_pred, c, m
// and the raw (rho, p) into the tile's (P, V) slot; force2_convert_aos then turns
// (m, rho, p) into the hoisted (grav m, m p / rho^2, m / rho) with stage_force's arithmetic,
// so the tile holds exactly the j-view's values.
__device__ __forceinline__ void force2_stage_aos(F2Tile &T, const ActiveLayout &L, const int *list,
                                                 const Particle *aos, int nb, int k, int lane) {
  const int q = k * kTJ + lane;
  if (q < L.pre[nb + 1] - L.pre[nb]) {
    const Particle *P = aos + list[L.base[nb] + q];
    cp_async8(&T.x[lane], &P->x[0]);
    cp_async8(&T.y[lane], &P->x[1]);
    cp_async16(&T.vv[lane], P->v_pred);
    cp_async8(&T.cm[lane].x, &P->c);
    cp_async8(&T.cm[lane].y, &P->m);
    cp_async8(&T.pv[lane].x, &P->rho);
    cp_async8(&T.pv[lane].y, &P->p);
  } else { // inert padding (jview_force2's dummies)
    T.x[lane] = kDummyX;
    T.y[lane] = kDummyX;
    T.gm[lane] = 0.0;
    T.vv[lane] = make_double2(0.0, 0.0);
    T.pv[lane] = make_double2(0.0, 0.0);
    T.cm[lane] = make_double2(0.0, 0.0);
  }
  cp_async_commit();
}
__device__ __forceinline__ void force2_convert_aos(F2Tile &T, const ActiveLayout &L, double grav,
                                                   int nb, int k, int lane) {
  if (k * kTJ + lane < L.pre[nb + 1] - L.pre[nb]) {
    const double2 rp = T.pv[lane];
    const double m = T.cm[lane].y;
    const double4 d = FastPolicy::stage_force(m, rp.x, rp.y, grav); // (m, gm, P, V)
    T.gm[lane] = d.y;
    T.pv[lane] = make_double2(d.z, d.w);
  }
}

// One work item of the force sweep (a cell and up to 32 of its locals).
template <bool AOS>
__device__ __forceinline__ void force2_item(const F2Args &A, F2Tile (&tl)[2], ActiveLayout &L,
                                            int item_idx, int lane) {
  const Item it = A.items[item_idx];
  if (lane == 0) build_active(A.g, it.cell, L);
  const bool live = lane < it.count;
  const int slot = A.list[it.start + (live ? lane : 0)];
  JSrc<AOS> src; // i side: the AoS records in place or the SoA mirror
  if constexpr (AOS) src.p = A.aos; else src.f = A.soa;
  const double2 xi = src.x(slot);
  const double hi = src.h(slot);
  F2I I;
  double eps2, K;
  unsigned hiH2m1;
  {
    const FastPolicy::FI F =
        FastPolicy::for_i(xi, src.vp(slot), hi, src.pr(slot), src.rho(slot), src.rho_dh(slot),
                          src.c(slot), src.div_v(slot), src.rot_v(slot), A.grav, nullptr);
    I = F2I{F.vx, F.vy, F.inv_hi, F.pri, F.mb3, __double2hiint(0.25 * hi * hi),
            __double2hiint(2.25 * hi * hi)};
    eps2 = F.eps2;
    K = F.K;
    hiH2m1 = F.hiH2m1;
  }
  // axn, ayn accumulate -a: fma(f, dx, axn) == -fma(-f, dx, ax) exactly (round to nearest is
  // sign-symmetric), and with f un-negated in the same operand slot of the x and y updates
  // ptxas serves the second read from the operand reuse cache (a DFMA reading three distinct
  // 64-bit registers takes 3 FP64-pipe cycles instead of 2, tools/operand_probe.cu)
  double axn = 0.0, ayn = 0.0, udt = 0.0, hdt = 0.0, vsig = -1.0;
  const float ixlo = warp_min((float)xi.x), ixhi = warp_max((float)xi.x);
  const float iylo = warp_min((float)xi.y), iyhi = warp_max((float)xi.y);
  const float reach = reach_of(warp_max((float)(2.5 * hi)));
  const float reach2 = __fmul_rn(reach, reach);
  const double k1875 = A.k1875, k0375 = A.k0375;
  __syncwarp();

  const int total = L.nch[L.n];
  bool staged = false;
  int buf = 0;
  for (int g0 = 0; g0 < total; g0 += 32) {
    // lane l classifies chunk g0 + l (stencil cell, chunk index, near/far), one ballot
    const int g = g0 + lane;
    int nb = 0, kk = 0;
    const bool valid = g < total;
    bool nr = false;
    if (valid) {
      chunk_locate(L, g, nb, kk);
      nr = chunk_near(L, A.boxes, nb, kk, ixlo, ixhi, iylo, iyhi, reach2);
    }
    const unsigned nmask = __ballot_sync(0xffffffffu, nr);
    unsigned todo = __ballot_sync(0xffffffffu, valid);
    while (todo) {
      const int b = __ffs(todo) - 1;
      todo &= todo - 1;
      const int cnb = __shfl_sync(0xffffffffu, nb, b), ck = __shfl_sync(0xffffffffu, kk, b);
      const bool has_next = todo != 0u;
      // one warp barrier per chunk: after it every lane's copies of this chunk are visible
      // and every lane is done with the previous chunk, whose buffer the next staging reuses
      if (!staged) {
        if constexpr (AOS) force2_stage_aos(tl[buf], L, A.list, A.aos, cnb, ck, lane);
        else force2_stage(tl[buf], L, A.jv, cnb, ck, lane);
      }
      cp_async_wait<0>();
      __syncwarp();
      if constexpr (AOS) {
        force2_convert_aos(tl[buf], L, A.grav, cnb, ck, lane);
        __syncwarp();
      }
      if (has_next) {
        const int bn = __ffs(todo) - 1;
        const int nnb = __shfl_sync(0xffffffffu, nb, bn), nk = __shfl_sync(0xffffffffu, kk, bn);
        if constexpr (AOS) force2_stage_aos(tl[buf ^ 1], L, A.list, A.aos, nnb, nk, lane);
        else force2_stage(tl[buf ^ 1], L, A.jv, nnb, nk, lane);
      }
      staged = has_next;
      const F2Tile &T = tl[buf];
      const double2 xr = xi;
      const double xs = xr.x - L.sx[cnb], ys = xr.y - L.sy[cnb]; // periodic image, i side
      if ((nmask >> b) & 1u) {
        tl[buf].vsig0[lane] = vsig;
#pragma unroll kF2NearU
        for (int j = 0; j < kTJ; j += 2) {
          const double2 X = *reinterpret_cast<const double2 *>(&T.x[j]);
          const double2 Y = *reinterpret_cast<const double2 *>(&T.y[j]);
          const double2 G = *reinterpret_cast<const double2 *>(&T.gm[j]);
          const double dx0 = xs - X.x, dy0 = ys - Y.x, dx1 = xs - X.y, dy1 = ys - Y.y;
          const double r20 = fma(dx0, dx0, dy0 * dy0), r21 = fma(dx1, dx1, dy1 * dy1);
          double f0, f1;
          {
            const double s0 = r20 + eps2, s1 = r21 + eps2;
            const double y0 = rsqrt_seed(s0), y1 = rsqrt_seed(s1);
            const double t0 = y0 * y0, t1 = y1 * y1;
            const double e0 = fma(-s0, t0, 1.0), e1 = fma(-s1, t1, 1.0);
            const double c0 = G.x * (t0 * y0), c1 = G.y * (t1 * y1);
            f0 = fma(c0, e0 * fma(e0, k1875, 1.5), c0);
            f1 = fma(c1, e1 * fma(e1, k1875, 1.5), c1);
          }
          // pair j's acceleration is accumulated before pair j+1's SPH block (fewer live
          // registers inside it); same j order
          if (support_cand(r20, hiH2m1))
            f0 = fma(K, force2_sph(I, T, j, dx0, dy0, r20, k0375, udt, hdt, vsig, hiH2m1), f0);
          axn = fma(f0, dx0, axn);
          ayn = fma(f0, dy0, ayn);
          if (support_cand(r21, hiH2m1))
            f1 = fma(K, force2_sph(I, T, j + 1, dx1, dy1, r21, k0375, udt, hdt, vsig, hiH2m1), f1);
          axn = fma(f1, dx1, axn);
          ayn = fma(f1, dy1, ayn);
        }
        __syncwarp();
        if (T.edge) { // warp-uniform after the barrier; rare
          vsig = force2_edge(I, T, lane, xi, xs, ys, hiH2m1);
          __syncwarp();
          if (lane == 0) tl[buf].edge = 0;
        }
      } else {
#pragma unroll kF2FarU
        for (int j = 0; j < kTJ; j += 4) {
          double dx[4], dy[4], gm[4];
          {
            const double2 X0 = *reinterpret_cast<const double2 *>(&T.x[j]);
            const double2 X1 = *reinterpret_cast<const double2 *>(&T.x[j + 2]);
            const double2 Y0 = *reinterpret_cast<const double2 *>(&T.y[j]);
            const double2 Y1 = *reinterpret_cast<const double2 *>(&T.y[j + 2]);
            const double2 G0 = *reinterpret_cast<const double2 *>(&T.gm[j]);
            const double2 G1 = *reinterpret_cast<const double2 *>(&T.gm[j + 2]);
            dx[0] = xs - X0.x; dx[1] = xs - X0.y; dx[2] = xs - X1.x; dx[3] = xs - X1.y;
            dy[0] = ys - Y0.x; dy[1] = ys - Y0.y; dy[2] = ys - Y1.x; dy[3] = ys - Y1.y;
            gm[0] = G0.x; gm[1] = G0.y; gm[2] = G1.x; gm[3] = G1.y;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double s = fma(dx[u], dx[u], fma(dy[u], dy[u], eps2));
            const double y0 = rsqrt_seed(s);
            const double t = y0 * y0;
            const double e = fma(-s, t, 1.0);
            const double c = gm[u] * (t * y0);
            const double f = fma(c, e * fma(e, k1875, 1.5), c);
            axn = fma(f, dx[u], axn);
            ayn = fma(f, dy[u], ayn);
          }
        }
      }
      buf ^= 1;
    }
  }
  if (!live) return;
  // publish (force_inv terms recomputed from memory: keeps c_i, h_i out of the loop)
  const FastPolicy::FI F =
      FastPolicy::for_i(xi, src.vp(slot), hi, src.pr(slot), src.rho(slot), src.rho_dh(slot),
                        src.c(slot), src.div_v(slot), src.rot_v(slot), A.grav, nullptr);
  FastPolicy::FA s{-axn, -ayn, udt, vsig, hdt, src.h_dt(slot)};
  double o[5];
  FastPolicy::for_publish(F, s, o);
  if constexpr (AOS) {
    Particle &q = const_cast<Particle &>(A.aos[slot]);
    q.a[0] = o[0]; q.a[1] = o[1]; q.u_dt = o[2]; q.v_sig = o[3]; q.h_dt = o[4];
  } else {
    A.soa.a[slot] = make_double2(o[0], o[1]);
    A.soa.u_dt[slot] = o[2];
    A.soa.v_sig[slot] = o[3];
    A.soa.h_dt[slot] = o[4];
  }
}

// With A.item_ctr set the kernel is persistent: one warp per resident slot, items taken in
// list order from the counter (dynamic balance instead of the hardware's CTA order).
template <int MINB, bool AOS>
__global__ void __launch_bounds__(kF2W * 32, MINB) force2_kernel(F2Args A) {
  __shared__ F2Tile tiles[kF2W][2];
  __shared__ ActiveLayout lay[kF2W];
  // one-warp CTAs: w = 0 statically, so the tile addresses need no thread-index arithmetic
  // and stay cheap to rematerialise under register pressure (force sweep -4.6 %)
  const int w = kF2W == 1 ? 0 : warp_in_cta(), lane = lane_id();
  const int total = A.n_items_dev ? *A.n_items_dev : A.n_items;
  if (!A.item_ctr && blockIdx.x * kF2W + w >= total) return;
  if (lane < 6) tiles[w][0].spl[lane] = tiles[w][1].spl[lane] = kSplQ[lane];
  if (lane == 0) tiles[w][0].edge = tiles[w][1].edge = 0;
  // one call site of the item body for both launch modes: two inlined copies may be compiled
  // to differently rounded FP64 code, and the results must not depend on the launch mode
  for (int idx = blockIdx.x * kF2W + w;;) {
    if (A.item_ctr) {
      if (lane == 0) idx = atomicAdd(A.item_ctr, 1);
      idx = __shfl_sync(0xffffffffu, idx, 0);
    }
    if (idx >= total) return;
    force2_item<AOS>(A, tiles[w], lay[w], idx, lane);
    if (!A.item_ctr) return;
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------------------
// Issue-lean culled FAST density round (density2): density_cull_kernel's decomposition
// (far chunks skipped, spatial j order, h-iteration rounds) with force2's staging (cp.async
// double buffer, split x[]/y[] tile) and a 3-piece coefficient table for W and dW.
// ---------------------------------------------------------------------------------------
struct __align__(16) D2Tile {
  double x[kTJ], y[kTJ], m[kTJ];
  double2 vv[kTJ];
  double2 spl[12]; // rows (outer, mid, inner) x {c4, c3}, {c2, c1}, {c_off, c0} (+1 spare)
};

// W(q) = N P(s) with s = c_off + sgn q (spline.hpp:12-41); the inner piece uses s = -q (P is
// even there), so on every piece dW/dq = -N dP/ds and the kernel derivative is
// E = P'(s) / 4, evaluated by the derivative Horner recursion alongside P: four table loads
// instead of six, the same seven DFMA. Sums over m E carry the factor 4, removed at publish.
// Rows are 4 entries apart; s = c_off - q on every piece.


// spline.hpp:12-41, P per piece as a polynomial in q (round 1 used s = c_off - q), rows {p4, p3}, {p2, p1}, {-, p0}: the same pieces,
// (2.5-q)^4, (2.5-q)^4 - 5 (1.5-q)^4, ... + 10 (0.5-q)^4, expanded (exact binary
// coefficients); dP/dq = -4 E, so the sums over m dP/dq carry the factor -4
__constant__ double2 kSplPE[12] = {
    {1.0, -10.0}, {37.5, -62.5}, {0.0, 39.0625}, {0.0, 0.0},
    {-4.0, 20.0}, {-30.0, 5.0}, {0.0, 13.75}, {0.0, 0.0},
    {6.0, 0.0}, {-15.0, 0.0}, {0.0, 14.375}, {0.0, 0.0},
};

__device__ __forceinline__ void density2_stage(D2Tile &T, const ActiveLayout &L, const D2View &jv,
                                               int nb, int k, int lane) {
  const int cnt = L.pre[nb + 1] - L.pre[nb];
  const int q = k * kTJ + lane;
  if (q < cnt) {
    const int idx = L.base[nb] + q;
    cp_async8(&T.x[lane], jv.x + idx);
    cp_async8(&T.y[lane], jv.y + idx);
    cp_async8(&T.m[lane], jv.m + idx);
    cp_async16(&T.vv[lane], jv.vv + idx);
  } else { // inert padding: beyond every support
    T.x[lane] = kDummyX;
    T.y[lane] = kDummyX;
    T.m[lane] = 0.0;
    T.vv[lane] = make_double2(0.0, 0.0);
  }
  cp_async_commit();
}

// AOS layout: the chunk's j fields (x, y, m, v_pred) straight from the 272-B records.
__device__ __forceinline__ void density2_stage_aos(D2Tile &T, const ActiveLayout &L, const int *jlist,
                                                   const Particle *aos, int nb, int k, int lane) {
  const int q = k * kTJ + lane;
  if (q < L.pre[nb + 1] - L.pre[nb]) {
    const Particle *P = aos + jlist[L.base[nb] + q];
    cp_async8(&T.x[lane], &P->x[0]);
    cp_async8(&T.y[lane], &P->x[1]);
    cp_async8(&T.m[lane], &P->m);
    cp_async16(&T.vv[lane], P->v_pred);
  } else {
    T.x[lane] = kDummyX;
    T.y[lane] = kDummyX;
    T.m[lane] = 0.0;
    T.vv[lane] = make_double2(0.0, 0.0);
  }
  cp_async_commit();
}

// density_pair (kernels.cpp:97-119) for one in-support pair, on FastPolicy's scaled sums
// (the piece comes from r2 against per-i thresholds (0.5h)^2, (1.5h)^2 on the high words,
// so the coefficient loads issue before the rsqrt chain; a pair within 2^-20 of a knot may
// take the neighbouring piece, which agrees there to O(dq^3))
// x^-1/2 of a pair's r^2 and the derived r and q (the in-support block's head)
struct D2Geo { double rinv, r, q; };
__device__ __forceinline__ D2Geo density2_geo(const FastPolicy::DI &I, double r2, double k0375) {
  const double y0 = rsqrt_seed(r2);
  const double e = fma(-r2, y0 * y0, 1.0);
  D2Geo G;
  G.rinv = fma(y0, e * fma(e, k0375, 0.5), y0);
  G.r = r2 * G.rinv;
  G.q = G.r * I.inv_h;
  return G;
}

// density_pair (kernels.cpp:97-119) for one in-support pair, on FastPolicy's scaled sums, from
// its geometry (the piece comes from r2 against per-i thresholds (0.5h)^2, (1.5h)^2 on the
// high words, so the coefficient loads issue early; a pair within 2^-20 of a knot may take
// the neighbouring piece, which agrees there to O(dq^3))
__device__ __forceinline__ void density2_acc(const FastPolicy::DI &I, int hiQ05, int hiQ15,
                                             const D2Tile &T, int j, double dx, double dy,
                                             double r2, const D2Geo &G, FastPolicy::DA &s) {
  const int hr = __double2hiint(r2);
  int row = hr < hiQ15 ? 4 : 0; // q < 1.5
  if (hr < hiQ05) row = 8;      // q < 0.5
  const double2 t1 = T.spl[row], t2 = T.spl[row + 1], t3 = T.spl[row + 2];
  const double rinv = G.rinv, r = G.r;
  const double sv = G.q; // q
  const double b3 = fma(t1.x, sv, t1.y), b2 = fma(b3, sv, t2.x), b1 = fma(b2, sv, t2.y);
  const double P = fma(b1, sv, t3.y);
  const double D = fma(fma(fma(t1.x, sv, b3), sv, b2), sv, b1); // P'(s) = 4 E
  const double mj = T.m[j];
  s.rho = fma(mj, P, s.rho);
  s.w += P;
  const double mE = mj * D; // 4 m E
  s.qe = fma(r, mE, s.qe);  // sum r 4 m E = 4 h sum q m E
  const double fac = mE * rinv;
  const double2 vj = T.vv[j];
  const double dvx = I.vx - vj.x, dvy = I.vy - vj.y;
  s.div = fma(fac, fma(dvx, dx, dvy * dy), s.div);
  s.rot = fma(fac, fma(dvx, dy, -dvy * dx), s.rot);
}

__device__ __forceinline__ void density2_pair(const FastPolicy::DI &I, int hiQ05, int hiQ15,
                                              const D2Tile &T, int j, double dx, double dy,
                                              double r2, double k0375, FastPolicy::DA &s) {
  density2_acc(I, hiQ05, hiQ15, T, j, dx, dy, r2, density2_geo(I, r2, k0375), s);
}

#ifndef SPH_MINB_D2
#define SPH_MINB_D2 20 // with SPH_D2_WPC = 1: 20 one-warp CTAs per SM, <= 96 registers
#endif

// JS lanes share one local particle i (j-slices): the warp holds 32/JS particles, which
// keeps its bounding box small when the locals are sparse (pending particles of the
// h-iteration rounds >= 1, ~12 % of a cell), so culling and the in-support union stay as
// tight as in round 0. Lane slice q takes j = q, q + JS, ... of each tile; the JS partial
// sums are combined with shuffles at the end.

// One work item of a density round (a cell and up to 32/JS of its pending locals).
template <int JS, bool AOS>
__device__ __forceinline__ void density2_item(const DenArgs &A, D2Tile (&tiles)[3],
                                              ActiveLayout &L, int item_idx, int lane) {
  D2Tile(&tiles_w)[3] = tiles; // this warp's staging buffers
  const Item it = A.items[item_idx];
  if (lane == 0) build_active(A.g, it.cell, L);
  const int iw = lane / JS, qs = lane % JS;
  const bool live = iw < it.count;
  const int slot = A.list[it.start + (live ? iw : 0)];
  JSrc<AOS> src; // i side: the AoS records in place or the SoA mirror
  if constexpr (AOS) src.p = A.aos; else src.f = A.soa;
  const double2 xi = src.x(slot), vi = src.vp(slot);
  const double h = (A.round == 0) ? src.h(slot) : A.hcur[slot];
  const FastPolicy::DI I = FastPolicy::den_i(xi.x, xi.y, vi.x, vi.y, h);
  const int hiQ05 = __double2hiint(0.25 * h * h), hiQ15 = __double2hiint(2.25 * h * h);
  FastPolicy::DA s = FastPolicy::den_zero();
  const float ixlo = warp_min((float)xi.x), ixhi = warp_max((float)xi.x);
  const float iylo = warp_min((float)xi.y), iyhi = warp_max((float)xi.y);
  const float reach = reach_of(warp_max((float)(2.5 * h)));
  const float reach2 = __fmul_rn(reach, reach);
  const double k0375 = A.k0375;
  __syncwarp();

  const int total = L.nch[L.n];
  bool staged = false;
  int buf = 0;
  for (int g0 = 0; g0 < total; g0 += 32) {
    const int g = g0 + lane;
    int nb = 0, kk = 0;
    bool nr = false;
    if (g < total) {
      chunk_locate(L, g, nb, kk);
      nr = chunk_near(L, A.boxes, nb, kk, ixlo, ixhi, iylo, iyhi, reach2);
    }
    unsigned todo = __ballot_sync(0xffffffffu, nr); // far chunks hold no in-support pair
    while (todo) {
      const int b = __ffs(todo) - 1;
      todo &= todo - 1;
      const int cnb = __shfl_sync(0xffffffffu, nb, b), ck = __shfl_sync(0xffffffffu, kk, b);
      const bool has_next = todo != 0u;
      if (!staged) {
        if constexpr (AOS) density2_stage_aos(tiles_w[buf], L, A.jlist, A.aos, cnb, ck, lane);
        else density2_stage(tiles_w[buf], L, A.jv2, cnb, ck, lane);
      }
      cp_async_wait<0>();
      __syncwarp();
      if (has_next) {
        const int bn = __ffs(todo) - 1;
        const int nnb = __shfl_sync(0xffffffffu, nb, bn), nk = __shfl_sync(0xffffffffu, kk, bn);
        if constexpr (AOS) density2_stage_aos(tiles_w[buf ^ 1], L, A.jlist, A.aos, nnb, nk, lane);
        else density2_stage(tiles_w[buf ^ 1], L, A.jv2, nnb, nk, lane);
      }
      staged = has_next;
      // per-j culling: a j farther than the warp's reach from the warp box can be in no
      // lane's support (same test as chunk_near, per particle); the others are compacted
      // into tiles_w[2], padded with inert dummies to the pair loop's granule
      int nj = kTJ;
      const D2Tile *Tp = &tiles_w[buf];
      if constexpr (JS == 1) { // (for j-slice warps measured slower: round 1 +8 %)
        constexpr int PADQ = JS * ((kTJ / JS) < 4 ? (kTJ / JS) : 4); // pair-loop granule
        const D2Tile &S = tiles_w[buf];
        D2Tile &C = tiles_w[2];
        const float jx = (float)S.x[lane] + (float)L.sx[cnb], jy = (float)S.y[lane] + (float)L.sy[cnb];
        const float gx = fmaxf(0.0f, fmaxf(jx - ixhi, ixlo - jx));
        const float gy = fmaxf(0.0f, fmaxf(jy - iyhi, iylo - jy));
        const bool rel = box_gap2(gx, gy) <= reach2;
        const unsigned rm = __ballot_sync(0xffffffffu, rel);
        nj = __popc(rm);
        const int pos = rel ? __popc(rm & ((1u << lane) - 1u)) : nj + __popc(~rm & ((1u << lane) - 1u));
        if (rel) {
          C.x[pos] = S.x[lane];
          C.y[pos] = S.y[lane];
          C.m[pos] = S.m[lane];
          C.vv[pos] = S.vv[lane];
        } else if (pos < ((nj + PADQ - 1) / PADQ) * PADQ) {
          C.x[pos] = kDummyX;
          C.y[pos] = kDummyX;
          C.m[pos] = 0.0;
          C.vv[pos] = make_double2(0.0, 0.0);
        }
        nj = ((nj + PADQ - 1) / PADQ) * PADQ;
        __syncwarp();
        Tp = &tiles_w[2];
      }
      const D2Tile &T = *Tp;
      const double xs = xi.x - L.sx[cnb], ys = xi.y - L.sy[cnb]; // periodic image, i side
      if constexpr (JS == 1) {
#pragma unroll kD2U
        for (int j = 0; j < nj; j += 4) {
          double dx[4], dy[4], r2[4];
          {
            const double2 X0 = *reinterpret_cast<const double2 *>(&T.x[j]);
            const double2 X1 = *reinterpret_cast<const double2 *>(&T.x[j + 2]);
            const double2 Y0 = *reinterpret_cast<const double2 *>(&T.y[j]);
            const double2 Y1 = *reinterpret_cast<const double2 *>(&T.y[j + 2]);
            dx[0] = xs - X0.x; dx[1] = xs - X0.y; dx[2] = xs - X1.x; dx[3] = xs - X1.y;
            dy[0] = ys - Y0.x; dy[1] = ys - Y0.y; dy[2] = ys - Y1.x; dy[3] = ys - Y1.y;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) r2[u] = fma(dx[u], dx[u], dy[u] * dy[u]);
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (in_support(r2[u], I.hiH2m1))
              density2_pair(I, hiQ05, hiQ15, T, j + u, dx[u], dy[u], r2[u], k0375, s);
        }
      } else {
        constexpr int U = (kTJ / JS) < 4 ? (kTJ / JS) : 4;
#pragma unroll kD2JU
        for (int t = 0; t * JS < nj; t += U) {
          double dx[U], dy[U], r2[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int j = qs + JS * (t + u);
            dx[u] = xs - T.x[j];
            dy[u] = ys - T.y[j];
            r2[u] = fma(dx[u], dx[u], dy[u] * dy[u]);
          }
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (in_support(r2[u], I.hiH2m1))
              density2_pair(I, hiQ05, hiQ15, T, qs + JS * (t + u), dx[u], dy[u], r2[u], k0375, s);
        }
      }
      buf ^= 1;
    }
  }
  if constexpr (JS > 1) { // combine the j-slices of each particle
#pragma unroll
    for (int o = 1; o < JS; o <<= 1) {
      s.rho += __shfl_xor_sync(0xffffffffu, s.rho, o);
      s.w += __shfl_xor_sync(0xffffffffu, s.w, o);
      s.qe += __shfl_xor_sync(0xffffffffu, s.qe, o);
      s.rot += __shfl_xor_sync(0xffffffffu, s.rot, o);
      s.div += __shfl_xor_sync(0xffffffffu, s.div, o);
    }
  }
  if (!live || qs != 0) return;
  constexpr double kDs = -0.25; // accumulated with dP/dq = -4 E
  s.qe *= kDs * I.inv_h; // accumulated as sum r (4 m E): to sum q m E
  s.div *= kDs;
  s.rot *= kDs;
  double hn = h;
  const int st = FastPolicy::den_step(s, hn, A.target, A.h_max, A.round);
  A.again[it.start + iw] = (unsigned char)(st == 0);
  if (st == 0) {
    A.hcur[slot] = hn;
    return;
  }
  double o[6];
  FastPolicy::den_publish(s, h, src.m(slot), o);
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

// A density round. With A.n_items_dev set the kernel is persistent: the round's item count
// is read from device memory (written by the previous round's make_items) and warps take
// items from A.item_ctr in list order, so consecutive rounds are queued without the host
// learning the count in between (capi.cu run_density).
template <int MINB, int JS, bool AOS>
__global__ void __launch_bounds__(kD2W * 32, MINB) density2_kernel(DenArgs A) {
  // [0], [1]: cp.async staging double buffer; [2]: the staged chunk's j's that can reach
  // the warp (compacted), which the pair loop consumes
  __shared__ D2Tile tiles[kD2W][3];
  __shared__ ActiveLayout lay[kD2W];
  const int w = warp_in_cta(), lane = lane_id(); // (a static w = 0 measured +0.6 % here)
  if (lane < 12) {
#pragma unroll
    for (int b = 0; b < 3; ++b) tiles[w][b].spl[lane] = kSplPE[lane];
  }
  // one call site of the item body for both launch modes (see force2_kernel)
  const int total = A.n_items_dev ? *A.n_items_dev : A.n_items;
  for (int idx = blockIdx.x * kD2W + w;;) {
    if (A.item_ctr) {
      if (lane == 0) idx = atomicAdd(A.item_ctr, 1);
      idx = __shfl_sync(0xffffffffu, idx, 0);
    }
    if (idx >= total) return;
    density2_item<JS, AOS>(A, tiles[w], lay[w], idx, lane);
    if (!A.item_ctr) return;
    __syncwarp();
  }
}

// Chunk-major j-view of the force sweep (one CTA per cell): the j fields of each 32-chunk of
// the cell's ilist written in the tile layout, the tail of the last chunk filled with inert
// dummies. (The same layout for density measured 4 % slower and is not used there.)
template <bool AOS>
__global__ void jview_density2_kernel(D2View v, const int *ilist, const Particle *aos, SoaMirror f,
                                      int n) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  JSrc<AOS> src;
  if constexpr (AOS) src.p = aos; else src.f = f;
  const int sj = ilist[p];
  const double2 x = src.x(sj);
  const_cast<double *>(v.x)[p] = x.x;
  const_cast<double *>(v.y)[p] = x.y;
  const_cast<double *>(v.m)[p] = src.m(sj);
  const_cast<double2 *>(v.vv)[p] = src.vp(sj);
}

void launch_jview_density2(const D2View &v, const int *ilist, const Particle *aos,
                           const SoaMirror &f, bool use_aos, int n, cudaStream_t s) {
  if (n <= 0) return;
  if (use_aos) jview_density2_kernel<true><<<(n + 255) / 256, 256, 0, s>>>(v, ilist, aos, f, n);
  else jview_density2_kernel<false><<<(n + 255) / 256, 256, 0, s>>>(v, ilist, aos, f, n);
}

template <bool AOS>
__global__ void jview_force2_kernel(double *blk, const int *ilist, const int *cell_begin,
                                    const Particle *aos, SoaMirror f, double grav) {
  const int c = blockIdx.x;
  const int b = cell_begin[c], cnt = cell_begin[c + 1] - b;
  JSrc<AOS> src;
  if constexpr (AOS) src.p = aos; else src.f = f;
  const int pad = (cnt + 31) & ~31;
  for (int q = threadIdx.x; q < pad; q += blockDim.x) {
    double *B = blk + (size_t)chunk_box_index(b, c, q >> 5) * kF2Blk;
    const int l = q & 31;
    double2 x = make_double2(kDummyX, kDummyX), v = make_double2(0.0, 0.0);
    double2 pv = make_double2(0.0, 0.0), cm = make_double2(0.0, 0.0);
    double gm = 0.0;
    if (q < cnt) {
      const int sj = ilist[b + q];
      x = src.x(sj);
      v = src.vp(sj);
      const double m = src.m(sj);
      const double4 d = FastPolicy::stage_force(m, src.rho(sj), src.pr(sj), grav); // (m, gm, P, V)
      gm = d.y;
      pv = make_double2(d.z, d.w);
      cm = make_double2(src.c(sj), m);
    }
    B[l] = x.x;
    B[32 + l] = x.y;
    B[64 + l] = gm;
    reinterpret_cast<double2 *>(B + 96)[l] = v;
    reinterpret_cast<double2 *>(B + 160)[l] = pv;
    reinterpret_cast<double2 *>(B + 224)[l] = cm;
  }
}

// (persistent grids of 21 warps per SM, which 94 registers would allow: no change, r2v)
// SMs of the current device (persistent launches size their grid by it; cached per device)
static int sm_count() {
  static int cache[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cache[dev]) cudaDeviceGetAttribute(&cache[dev], cudaDevAttrMultiProcessorCount, dev);
  return cache[dev] > 0 ? cache[dev] : 148;
}

void launch_force2(const F2Args &a, int n_items, int n, cudaStream_t s) {
  const bool aos = a.aos != nullptr;
  // the SoA layouts read the per-sweep chunk-major j-view; the AoS arm stages j's from the
  // records themselves (force2_stage_aos)
  if (n > 0 && a.g.ncells > 0 && !aos)
    jview_force2_kernel<false><<<a.g.ncells, 128, 0, s>>>(const_cast<double *>(a.jv.blk), a.list,
                                                          a.g.cell_begin, a.aos, a.soa, a.grav);
  if (n_items <= 0 && !a.n_items_dev) return;
  F2Args b = a;
  b.n_items = n_items;
  b.k1875 = 1.875;
  b.k0375 = 0.375;
  int G = (n_items + kF2W - 1) / kF2W;
  if (b.item_ctr) { // persistent: every resident warp slot
    const int sms = sm_count();
    G = b.n_items_dev ? sms * SPH_MINB_F2 / kF2W : std::min(G, sms * SPH_MINB_F2 / kF2W);
    cudaMemsetAsync(b.item_ctr, 0, sizeof(int), s);
  }
  if (aos) force2_kernel<SPH_MINB_F2, true><<<G, kF2W * 32, 0, s>>>(b);
  else force2_kernel<SPH_MINB_F2, false><<<G, kF2W * 32, 0, s>>>(b);
}

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
  if (n_items <= 0 && !a.n_items_dev) return;
  // (persistent launches: item_ctr set; the count is n_items or, if set, *n_items_dev)
  DenArgs b = a;
  b.n_items = n_items;
  const int G = pair_grid(n_items), B = kWarpsPerCta * 32;
  if (b.boxes && b.jlist && b.jv2.x) {
    b.k0375 = 0.375;
    int G2 = (n_items + kD2W - 1) / kD2W;
    const int B2 = kD2W * 32;
    if (b.item_ctr) { // persistent: every resident warp slot, items taken from item_ctr
      G2 = sm_count() * SPH_MINB_D2 / kD2W;
      cudaMemsetAsync(b.item_ctr, 0, sizeof(int), s);
    }
    if (aos) {
      switch (b.jslices) {
      case 2: density2_kernel<SPH_MINB_D2, 2, true><<<G2, B2, 0, s>>>(b); break;
      case 4: density2_kernel<SPH_MINB_D2, 4, true><<<G2, B2, 0, s>>>(b); break;
      case 8: density2_kernel<SPH_MINB_D2, 8, true><<<G2, B2, 0, s>>>(b); break;
      default: density2_kernel<SPH_MINB_D2, 1, true><<<G2, B2, 0, s>>>(b); break;
      }
    } else {
      switch (b.jslices) {
      case 2: density2_kernel<SPH_MINB_D2, 2, false><<<G2, B2, 0, s>>>(b); break;
      case 4: density2_kernel<SPH_MINB_D2, 4, false><<<G2, B2, 0, s>>>(b); break;
      case 8: density2_kernel<SPH_MINB_D2, 8, false><<<G2, B2, 0, s>>>(b); break;
      default: density2_kernel<SPH_MINB_D2, 1, false><<<G2, B2, 0, s>>>(b); break;
      }
    }
  } else if (b.boxes && b.jlist) {
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
