/* sph_oracle.c — TEST INFRASTRUCTURE: CPU restatement of the reference SPH hot path.
 *
 * This is the parity oracle, not product code. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it, and only as the checker (or the CPU
 * baseline). It restates, in plain C, the reference algorithm of
 *   /root/reference/proj/include/soaview/sph/spline.hpp:8-41   (M5 spline)
 *   /root/reference/proj/src/sph/kernels.cpp:24               (min image)
 *   /root/reference/proj/src/sph/kernels.cpp:97-202           (pair fns, h-step, publish)
 *   /root/reference/proj/src/sph/kernels.cpp:204-303          (per-cell nests)
 *   /root/reference/proj/src/sph/kernels.cpp:305-341          (drift / kick lanes)
 *   /root/reference/proj/src/sph/grid.cpp:15-26, 31-54, 76-184 (RNG map, nx, target, IC, grid)
 * with the same operation order and no FMA contraction (built with -ffp-contract=off,
 * like the reference, src/CMakeLists.txt:21-22), so results are bit-identical to the
 * reference. Parity of this restatement is PINNED against the reference itself
 * (oracle/_ref, compiled from /root/reference by oracle/Makefile) and against the
 * committed golden vectors in tests/golden/ (made by tests/golden/make_golden.py).
 *
 * Path (AoS/SoA view), Order (local-active/active-local) and Guard (branch/mask) are
 * bitwise-equivalent in the reference (test_sph.cpp:308-337), so one restatement
 * covers every variant.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  double x[2], v[2], v_pred[2], a[2];
  double m, rho, p, u, u_pred, u_dt, c, h, wcount, rho_dh, rot_v, div_v, v_sig, h_dt, dt_next;
  int32_t frozen, moved;
  int64_t id, cell, flags;
  double dbg[2], spare[5];
} orc_particle; /* particle.hpp:11-38, 272 bytes */

_Static_assert(sizeof(orc_particle) == 272, "record must be 272 bytes");

#define SUPPORT 2.5                   /* spline.hpp:8 */
#define NORM2D 0.025486029252413597   /* spline.hpp:9 */

/* spline.hpp:12-25 */
double orc_kernel_w(double q) {
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
  return NORM2D * acc;
}

/* spline.hpp:28-41 */
double orc_kernel_dw(double q) {
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
  return NORM2D * -4.0 * acc;
}

static inline double min_image(double d) { return d - round(d); } /* kernels.cpp:24 */
static inline double dmin(double a, double b) { return (b < a) ? b : a; } /* std::min */
static inline double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */

/* grid.cpp:23-26 */
int orc_grid_nx(int64_t n, int ppc) {
  double cell = sqrt((double)ppc / (double)(n > 1 ? n : 1));
  int v = (int)floor(1.0 / cell);
  return v > 1 ? v : 1;
}

static inline int clamp_cell(int v, int n) { return v < 0 ? 0 : (v > n - 1 ? n - 1 : v); }

/* Deduplicated, wrapped 3x3 stencil in (dy, dx) row-major order, grid.cpp:161-176. */
static int stencil(int c, int nx, int ny, int *idx) {
  int cy = c / nx, cx = c % nx, n = 0;
  for (int dy = -1; dy <= 1; ++dy)
    for (int dx = -1; dx <= 1; ++dx) {
      int wy = (cy + dy + ny) % ny, wx = (cx + dx + nx) % nx, ci = wy * nx + wx, seen = 0;
      for (int k = 0; k < n; ++k)
        if (idx[k] == ci) seen = 1;
      if (!seen) idx[n++] = ci;
    }
  return n;
}

/* build_grid (grid.cpp:145-158): cell = clamp(floor(x*nx)); local lists in `recs` order.
 * Writes p->cell; fills cell_begin[ncells+1] and local_idx[n] (indices into recs). */
void orc_build_grid(orc_particle *recs, int64_t n, int nx, int ny, int64_t *cell_begin,
                    int64_t *local_idx) {
  int nc = nx * ny;
  int64_t *cnt = (int64_t *)calloc((size_t)nc + 1, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) {
    orc_particle *p = &recs[i];
    int cx = clamp_cell((int)floor(p->x[0] * nx), nx);
    int cy = clamp_cell((int)floor(p->x[1] * nx), ny);
    int ci = cy * nx + cx;
    p->cell = ci;
    cnt[ci + 1]++;
  }
  for (int c = 0; c < nc; ++c) cnt[c + 1] += cnt[c];
  memcpy(cell_begin, cnt, sizeof(int64_t) * ((size_t)nc + 1));
  for (int64_t i = 0; i < n; ++i) local_idx[cnt[recs[i].cell]++] = i;
  free(cnt);
}

typedef struct {
  orc_particle *recs;
  int nx, ny;
  double cell_size;
  const int64_t *cb, *li;
} grid_t;

/* Active list of cell c as a flat index array (concatenated stencil cells). */
static int64_t active_of(const grid_t *g, int c, int64_t *out) {
  int idx[9], nn = stencil(c, g->nx, g->ny, idx);
  int64_t k = 0;
  for (int s = 0; s < nn; ++s)
    for (int64_t t = g->cb[idx[s]]; t < g->cb[idx[s] + 1]; ++t) out[k++] = g->li[t];
  return k;
}

static int64_t max_active(const grid_t *g) {
  int64_t m = 0;
  for (int c = 0; c < g->nx * g->ny; ++c) {
    int idx[9], nn = stencil(c, g->nx, g->ny, idx);
    int64_t k = 0;
    for (int s = 0; s < nn; ++s) k += g->cb[idx[s] + 1] - g->cb[idx[s]];
    if (k > m) m = k;
  }
  return m;
}

typedef struct { double rho, wcount, rho_dh, rot_v, div_v; } dacc_t; /* kernels.cpp:69-75 */

/* kernels.cpp:97-119 (branch guard; mask is bitwise-identical) */
static inline void density_pair(double xi0, double xi1, double vi0, double vi1, double inv_h,
                                const orc_particle *pj, dacc_t *s) {
  double dx0 = min_image(xi0 - pj->x[0]);
  double dx1 = min_image(xi1 - pj->x[1]);
  double r2 = dx0 * dx0 + dx1 * dx1;
  if (r2 <= 0.0) return;
  double r = sqrt(r2);
  double q = r * inv_h;
  if (!(q < SUPPORT)) return;
  double mj = pj->m;
  double w = orc_kernel_w(q);
  double dw = orc_kernel_dw(q);
  s->rho += mj * w;
  s->wcount += w;
  s->rho_dh -= mj * (2.0 * w + q * dw);
  double dv0 = vi0 - pj->v_pred[0];
  double dv1 = vi1 - pj->v_pred[1];
  double fac = mj * dw / r;
  s->div_v -= fac * (dv0 * dx0 + dv1 * dx1);
  s->rot_v += fac * (dv0 * dx1 - dv1 * dx0);
}

/* density_step, kernels.cpp:184-192. returns 0 Again, 1 Done, 2 Fail; *h updated. */
static inline int density_step(const dacc_t *s, double *h, double target, double h_max,
                               int iter) {
  double wc = s->wcount + orc_kernel_w(0.0);
  double ratio = sqrt(target / wc);
  if (fabs(ratio - 1.0) < 1.0e-4) return 1;
  double hn = dmin(h_max, *h * dmin(1.2, dmax(0.8, ratio)));
  if (hn == *h) return 1;
  if (iter >= 29) return 2;
  *h = hn;
  return 0;
}

/* density_cell_la, kernels.cpp:204-227 + density_publish :194-202.
 * rounds_out (optional, indexed like recs) receives the number of h-rounds. */
static void density_cell(const grid_t *g, int c, const int64_t *act, int64_t na, double target,
                         double h_max, int32_t *rounds_out) {
  for (int64_t t = g->cb[c]; t < g->cb[c + 1]; ++t) {
    orc_particle *pi = &g->recs[g->li[t]];
    double xi0 = pi->x[0], xi1 = pi->x[1], vi0 = pi->v_pred[0], vi1 = pi->v_pred[1];
    double mi = pi->m, h = pi->h;
    dacc_t s;
    int iter;
    for (iter = 0;; ++iter) {
      memset(&s, 0, sizeof s);
      double inv_h = 1.0 / h;
      for (int64_t j = 0; j < na; ++j)
        density_pair(xi0, xi1, vi0, vi1, inv_h, &g->recs[act[j]], &s);
      int st = density_step(&s, &h, target, h_max, iter);
      if (st == 0) continue;
      if (st == 2) pi->flags += 1;
      break;
    }
    if (rounds_out) rounds_out[g->li[t]] = iter + 1;
    double w0 = orc_kernel_w(0.0);
    double inv_h = 1.0 / h;
    double inv_h2 = inv_h * inv_h;
    double inv_h3 = inv_h2 * inv_h;
    pi->h = h;
    pi->rho = (s.rho + mi * w0) * inv_h2;
    pi->wcount = s.wcount + w0;
    pi->rho_dh = (s.rho_dh - 2.0 * mi * w0) * inv_h3;
    pi->rot_v = s.rot_v * inv_h3;
    pi->div_v = s.div_v * inv_h3;
  }
}

typedef struct { double x0, x1, v0, v1, hi, inv_hi, inv_hi3, pri, bi, eps2, ci; } finv_t;
typedef struct { double a0, a1, udt, vsig, hdt; } facc_t;

/* force_inv, kernels.cpp:155-172 */
static inline finv_t force_inv(const orc_particle *p) {
  finv_t I;
  I.x0 = p->x[0];
  I.x1 = p->x[1];
  I.v0 = p->v_pred[0];
  I.v1 = p->v_pred[1];
  I.hi = p->h;
  I.inv_hi = 1.0 / I.hi;
  I.inv_hi3 = I.inv_hi * I.inv_hi * I.inv_hi;
  double rhoi = p->rho;
  I.pri = p->p / (rhoi * rhoi) * (1.0 + 0.5 * I.hi * p->rho_dh / rhoi);
  double adiv = fabs(p->div_v);
  I.ci = p->c;
  I.bi = adiv / (adiv + fabs(p->rot_v) + 0.0001 * I.ci * I.inv_hi);
  I.eps2 = 0.01 * I.hi * I.hi;
  return I;
}

/* force_pair, kernels.cpp:121-153 (branch guard) */
static inline void force_pair(const finv_t *I, double grav, const orc_particle *pj, facc_t *s) {
  double dx0 = min_image(I->x0 - pj->x[0]);
  double dx1 = min_image(I->x1 - pj->x[1]);
  double r2 = dx0 * dx0 + dx1 * dx1;
  if (r2 <= 0.0) return;
  double mj = pj->m;
  double soft = r2 + I->eps2;
  double gfac = grav * mj / (soft * sqrt(soft));
  s->a0 -= gfac * dx0;
  s->a1 -= gfac * dx1;
  double r = sqrt(r2);
  double q = r * I->inv_hi;
  if (!(q < SUPPORT)) return;
  double rhoj = pj->rho;
  double dwi = orc_kernel_dw(q) * I->inv_hi3;
  double inv_r = 1.0 / r;
  double prj = pj->p / (rhoj * rhoj);
  double acc = mj * (I->pri + prj) * dwi * inv_r;
  s->a0 -= acc * dx0;
  s->a1 -= acc * dx1;
  double dv0 = I->v0 - pj->v_pred[0];
  double dv1 = I->v1 - pj->v_pred[1];
  double dvdr = dv0 * dx0 + dv1 * dx1;
  s->udt += mj * I->pri * dwi * dvdr * inv_r;
  double mu = dmin(0.0, dvdr * inv_r);
  s->vsig = dmax(s->vsig, 1.0 * (I->ci + pj->c - 3.0 * mu * I->bi));
  s->hdt -= mj / rhoj * dvdr * inv_r * dwi * 0.5 * I->hi;
}

/* force_cell_la, kernels.cpp:273-284 + AosRecs::store :369-376 */
static void force_cell(const grid_t *g, int c, const int64_t *act, int64_t na, double grav) {
  for (int64_t t = g->cb[c]; t < g->cb[c + 1]; ++t) {
    orc_particle *pi = &g->recs[g->li[t]];
    finv_t I = force_inv(pi);
    facc_t s = {0.0, 0.0, 0.0, 0.0, pi->h_dt};
    for (int64_t j = 0; j < na; ++j) force_pair(&I, grav, &g->recs[act[j]], &s);
    pi->a[0] = s.a0;
    pi->a[1] = s.a1;
    pi->u_dt = s.udt;
    pi->v_sig = s.vsig;
    pi->h_dt = s.hdt;
  }
}

/* drift_lane / drift_one, kernels.cpp:305-312, :880-883 */
void orc_drift_one(orc_particle *p, const double *par5) {
  double dt = par5[0];
  double adv = p->frozen ? 0.0 : dt;
  p->x[0] += adv * p->v_pred[0];
  p->x[1] += adv * p->v_pred[1];
  p->u_pred = p->u + 0.5 * adv * p->u_dt;
  p->moved = p->frozen ? 0 : 1;
}

/* kick1_lane / kick1_one, kernels.cpp:314-323, :885-887 */
void orc_kick1_one(orc_particle *p, const double *par5) {
  double half = 0.5 * par5[0];
  p->v[0] += half * p->a[0];
  p->v[1] += half * p->a[1];
  p->u += half * p->u_dt;
  double vn = sqrt(p->v[0] * p->v[0] + p->v[1] * p->v[1]);
  double an = sqrt(p->a[0] * p->a[0] + p->a[1] * p->a[1]);
  p->dt_next = dmin(0.005 / (vn + 1.0e-12), sqrt(0.005 / (an + 1.0e-12)));
}

/* kick2_lane / kick2_one, kernels.cpp:325-341, :889-893 */
void orc_kick2_one(orc_particle *p, const double *par5) {
  double dt = par5[0], gamma = par5[1], cfl = par5[2];
  double half = 0.5 * dt;
  p->v[0] += half * p->a[0];
  p->v[1] += half * p->a[1];
  p->u += half * (p->u_dt + p->dbg[0]);
  if (p->u < 0.5 * p->u_pred) p->u = 0.5 * p->u_pred;
  p->v_pred[0] = p->v[0];
  p->v_pred[1] = p->v[1];
  p->u_pred = p->u;
  p->c = sqrt(gamma * (gamma - 1.0) * dmax(p->u, 1.0e-12));
  p->p = (gamma - 1.0) * p->rho * p->u;
  p->dt_next = dmin(p->dt_next, cfl * p->h / dmax(p->v_sig, p->c + p->c));
  p->h_dt = 0.0;
}

/* One sweep of kernel k over all cells, or over the cells with cell_mask[c] != 0 (the owned
 * cells of a domain-decomposition rank; other cells still feed the active lists)
 * (run_sweep, kernels.cpp:861-872).
 * kernel: 0 density, 1 force, 2 drift, 3 kick1, 4 kick2 (KernelId order, kernels.hpp:9).
 * rounds_out: optional per-record h-round counts (density only). Returns 0. */
int orc_sweep_masked(int kernel, orc_particle *recs, int nx, int ny, double cell_size,
                     const int64_t *cell_begin, const int64_t *local_idx, const double *par5,
                     int threads, int32_t *rounds_out, const uint8_t *cell_mask) {
  grid_t g = {recs, nx, ny, cell_size, cell_begin, local_idx};
  int nc = nx * ny;
  if (kernel >= 2) {
#pragma omp parallel for schedule(dynamic, 16) num_threads(threads > 0 ? threads : 1)
    for (int c = 0; c < nc; ++c) {
      if (cell_mask && !cell_mask[c]) continue;
      for (int64_t t = cell_begin[c]; t < cell_begin[c + 1]; ++t) {
      orc_particle *p = &recs[local_idx[t]];
      if (kernel == 2) orc_drift_one(p, par5);
      else if (kernel == 3) orc_kick1_one(p, par5);
      else orc_kick2_one(p, par5);
      }
    }
    return 0;
  }
  int64_t cap = max_active(&g);
  double target = par5[4], grav = par5[3];
  double h_max = cell_size / SUPPORT; /* kernels.cpp:542 */
#pragma omp parallel num_threads(threads > 0 ? threads : 1)
  {
    int64_t *act = (int64_t *)malloc(sizeof(int64_t) * (size_t)(cap > 0 ? cap : 1));
#pragma omp for schedule(dynamic, 1)
    for (int c = 0; c < nc; ++c) {
      if (cell_begin[c + 1] == cell_begin[c]) continue; /* kernels.cpp:548 */
      if (cell_mask && !cell_mask[c]) continue;         /* not owned (decomposition) */
      int64_t na = active_of(&g, c, act);
      if (kernel == 0) density_cell(&g, c, act, na, target, h_max, rounds_out);
      else force_cell(&g, c, act, na, grav);
    }
    free(act);
  }
  return 0;
}

int orc_sweep(int kernel, orc_particle *recs, int nx, int ny, double cell_size,
              const int64_t *cell_begin, const int64_t *local_idx, const double *par5,
              int threads, int32_t *rounds_out) {
  return orc_sweep_masked(kernel, recs, nx, ny, cell_size, cell_begin, local_idx, par5, threads,
                          rounds_out, NULL);
}

/* mean_wcount, grid.cpp:31-54: per-particle sums in parallel, total summed in order. */
double orc_mean_wcount(orc_particle *recs, int nx, int ny, const int64_t *cell_begin,
                       const int64_t *local_idx, int threads) {
  grid_t g = {recs, nx, ny, 0.0, cell_begin, local_idx};
  int nc = nx * ny;
  int64_t n = cell_begin[nc];
  double *wc = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  int64_t cap = max_active(&g);
  const double w0 = orc_kernel_w(0.0);
#pragma omp parallel num_threads(threads > 0 ? threads : 1)
  {
    int64_t *act = (int64_t *)malloc(sizeof(int64_t) * (size_t)(cap > 0 ? cap : 1));
#pragma omp for schedule(dynamic, 1)
    for (int c = 0; c < nc; ++c) {
      int64_t na = active_of(&g, c, act);
      for (int64_t t = cell_begin[c]; t < cell_begin[c + 1]; ++t) {
        const orc_particle *pi = &recs[local_idx[t]];
        double w = w0, inv_h = 1.0 / pi->h;
        for (int64_t j = 0; j < na; ++j) {
          const orc_particle *pj = &recs[act[j]];
          double dx0 = pi->x[0] - pj->x[0];
          double dx1 = pi->x[1] - pj->x[1];
          dx0 -= round(dx0);
          dx1 -= round(dx1);
          double r2 = dx0 * dx0 + dx1 * dx1;
          if (r2 <= 0.0) continue;
          double q = sqrt(r2) * inv_h;
          if (q < SUPPORT) w += orc_kernel_w(q);
        }
        wc[t] = w;
      }
    }
    free(act);
  }
  double total = 0.0;
  for (int64_t t = 0; t < n; ++t) total += wc[t];
  free(wc);
  return n ? total / (double)n : 0.0;
}

/* std::mt19937_64 (published MT19937-64 algorithm; parameters of [rand.predef]). */
typedef struct { uint64_t mt[312]; int mti; } mt64_t;
static void mt64_seed(mt64_t *s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->mti = 312;
}
static uint64_t mt64_next(mt64_t *s) {
  static const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (s->mti >= 312) {
    int i;
    uint64_t x;
    for (i = 0; i < 312 - 156; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    for (; i < 311; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + (156 - 312)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    x = (s->mt[311] & UM) | (s->mt[0] & LM);
    s->mt[311] = s->mt[155] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    s->mti = 0;
  }
  uint64_t x = s->mt[s->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}
static inline double unit_real(mt64_t *s) { return (double)(mt64_next(s) >> 11) * 0x1.0p-53; } /* grid.cpp:15-19 */

/* Proto records of make_particles (grid.cpp:77-98), in id order.
 * kind 0: the reference IC (uniform random positions).
 * kind 1: builder-defined clustered IC for variable ppc (BASELINE config 3; the reference
 *         has no such generator): the same RNG stream, half the particles uniform, half in
 *         16 Gaussian clumps (sigma = 1 cell) whose centres are drawn first; the normal
 *         deviates are Irwin-Hall sums of 12 unit_real draws minus 6 (exact double
 *         arithmetic, no libm) and positions wrap with x - floor(x). All other fields as
 *         the reference. */
void orc_make_proto_kind(int64_t n, int ppc, uint64_t seed, int kind, orc_particle *out) {
  mt64_t rng;
  mt64_seed(&rng, seed);
  if (n < 1) n = 1;
  double cell_size = 1.0 / orc_grid_nx(n, ppc);
  double h_warm = 0.8 * cell_size / SUPPORT;
  double ccx[16], ccy[16];
  const double sigma = 1.0 * cell_size;
  if (kind == 1)
    for (int k = 0; k < 16; ++k) {
      ccx[k] = unit_real(&rng);
      ccy[k] = unit_real(&rng);
    }
  for (int64_t i = 0; i < n; ++i) {
    orc_particle *p = &out[i];
    memset(p, 0, sizeof *p);
    if (kind == 1 && i >= n / 2) {
      int k = (int)(mt64_next(&rng) % 16u);
      double gx = 0.0, gy = 0.0;
      for (int t = 0; t < 12; ++t) gx += unit_real(&rng);
      for (int t = 0; t < 12; ++t) gy += unit_real(&rng);
      double x0 = ccx[k] + sigma * (gx - 6.0);
      double x1 = ccy[k] + sigma * (gy - 6.0);
      p->x[0] = x0 - floor(x0);
      p->x[1] = x1 - floor(x1);
    } else {
      p->x[0] = unit_real(&rng);
      p->x[1] = unit_real(&rng);
    }
    p->v[0] = (unit_real(&rng) * 2.0 - 1.0) * 0.05;
    p->v[1] = (unit_real(&rng) * 2.0 - 1.0) * 0.05;
    p->v_pred[0] = p->v[0];
    p->v_pred[1] = p->v[1];
    p->u = 0.5 + unit_real(&rng);
    p->u_pred = p->u;
    p->m = 1.0 / (double)n;
    p->h = h_warm;
    p->dt_next = 1.0e30;
    p->id = i;
  }
}

void orc_make_proto(int64_t n, int ppc, uint64_t seed, orc_particle *out) {
  orc_make_proto_kind(n, ppc, seed, 0, out);
}

static int g_sort_nx;
static int cell_of(const orc_particle *p) {
  int cx = clamp_cell((int)floor(p->x[0] * g_sort_nx), g_sort_nx);
  int cy = clamp_cell((int)floor(p->x[1] * g_sort_nx), g_sort_nx);
  return cy * g_sort_nx + cx;
}
static int cmp_cell_id(const void *a, const void *b) {
  const orc_particle *pa = (const orc_particle *)a, *pb = (const orc_particle *)b;
  int ca = cell_of(pa), cb = cell_of(pb);
  if (ca != cb) return ca < cb ? -1 : 1;
  return pa->id < pb->id ? -1 : (pa->id > pb->id ? 1 : 0);
}

/* make_particles (grid.cpp:76-143), continuous layout: `out` (n records) receives the
 * store.all order = sorted by (cell, id) (grid.cpp:117-132); par5 receives SphParams
 * defaults with the calibrated target_wcount. Values are layout-independent
 * (test_sph.cpp:138-149), so this also pins the scattered layout by id. */
int orc_make_particles_kind(int64_t n, int ppc, uint64_t seed, int kind, orc_particle *out,
                            double *par5, int threads) {
  if (n < 1) n = 1;
  orc_make_proto_kind(n, ppc, seed, kind, out);
  int nx = orc_grid_nx(n, ppc);
  g_sort_nx = nx;
  qsort(out, (size_t)n, sizeof(orc_particle), cmp_cell_id);
  int nc = nx * nx;
  int64_t *cb = (int64_t *)malloc(sizeof(int64_t) * ((size_t)nc + 1));
  int64_t *li = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  orc_build_grid(out, n, nx, nx, cb, li);
  par5[0] = 1.0e-4;
  par5[1] = 5.0 / 3.0;
  par5[2] = 0.1;
  par5[3] = 1.0;
  par5[4] = orc_mean_wcount(out, nx, nx, cb, li, threads);
  double cell_size = 1.0 / nx;
  orc_sweep(0, out, nx, nx, cell_size, cb, li, par5, threads, NULL);
  for (int64_t i = 0; i < n; ++i) {
    orc_particle *p = &out[i];
    p->p = (par5[1] - 1.0) * p->rho * p->u;
    p->c = sqrt(par5[1] * (par5[1] - 1.0) * p->u);
  }
  orc_sweep(1, out, nx, nx, cell_size, cb, li, par5, threads, NULL);
  free(cb);
  free(li);
  return 0;
}

int orc_make_particles(int64_t n, int ppc, uint64_t seed, orc_particle *out, double *par5,
                       int threads) {
  return orc_make_particles_kind(n, ppc, seed, 0, out, par5, threads);
}

/* Pair statistics of one density round at the records' current h:
 * counts of active pairs, pairs with r2 > 0, and pairs with q < 2.5 / 1.5 / 0.5, over the
 * cells with cell_mask[c] != 0 (all cells when cell_mask is NULL). */
void orc_pair_stats(orc_particle *recs, int nx, int ny, const int64_t *cell_begin,
                    const int64_t *local_idx, const uint8_t *cell_mask, int threads,
                    int64_t *out5) {
  grid_t g = {recs, nx, ny, 0.0, cell_begin, local_idx};
  int nc = nx * ny;
  int64_t cap = max_active(&g);
  int64_t tot[5] = {0, 0, 0, 0, 0};
#pragma omp parallel num_threads(threads > 0 ? threads : 1)
  {
    int64_t loc[5] = {0, 0, 0, 0, 0};
    int64_t *act = (int64_t *)malloc(sizeof(int64_t) * (size_t)(cap > 0 ? cap : 1));
#pragma omp for schedule(dynamic, 1)
    for (int c = 0; c < nc; ++c) {
      if (cell_mask && !cell_mask[c]) continue;
      int64_t na = active_of(&g, c, act);
      for (int64_t t = cell_begin[c]; t < cell_begin[c + 1]; ++t) {
        const orc_particle *pi = &recs[local_idx[t]];
        double inv_h = 1.0 / pi->h;
        for (int64_t j = 0; j < na; ++j) {
          const orc_particle *pj = &recs[act[j]];
          double dx0 = min_image(pi->x[0] - pj->x[0]);
          double dx1 = min_image(pi->x[1] - pj->x[1]);
          double r2 = dx0 * dx0 + dx1 * dx1;
          loc[0]++;
          if (r2 <= 0.0) continue;
          loc[1]++;
          double q = sqrt(r2) * inv_h;
          if (q < 2.5) loc[2]++;
          if (q < 1.5) loc[3]++;
          if (q < 0.5) loc[4]++;
        }
      }
    }
    free(act);
#pragma omp critical
    for (int k = 0; k < 5; ++k) tot[k] += loc[k];
  }
  for (int k = 0; k < 5; ++k) out5[k] = tot[k];
}

/* orc_pair_stats for one cell c over every i_stride-th local particle, threads splitting the
 * locals (a bounded sample of a dense cell; the counts are of the sampled pairs). */
void orc_pair_stats_cell(orc_particle *recs, int nx, int ny, const int64_t *cell_begin,
                         const int64_t *local_idx, int c, int64_t i_stride, int threads,
                         int64_t *out5) {
  grid_t g = {recs, nx, ny, 0.0, cell_begin, local_idx};
  int64_t cap = max_active(&g);
  int64_t *act = (int64_t *)malloc(sizeof(int64_t) * (size_t)(cap > 0 ? cap : 1));
  int64_t na = active_of(&g, c, act);
  if (i_stride < 1) i_stride = 1;
  int64_t b = cell_begin[c], nsel = (cell_begin[c + 1] - b + i_stride - 1) / i_stride;
  int64_t tot[5] = {0, 0, 0, 0, 0};
#pragma omp parallel num_threads(threads > 0 ? threads : 1)
  {
    int64_t loc[5] = {0, 0, 0, 0, 0};
#pragma omp for schedule(dynamic, 4)
    for (int64_t k = 0; k < nsel; ++k) {
      const orc_particle *pi = &recs[local_idx[b + k * i_stride]];
      double inv_h = 1.0 / pi->h;
      for (int64_t j = 0; j < na; ++j) {
        const orc_particle *pj = &recs[act[j]];
        double dx0 = min_image(pi->x[0] - pj->x[0]);
        double dx1 = min_image(pi->x[1] - pj->x[1]);
        double r2 = dx0 * dx0 + dx1 * dx1;
        loc[0]++;
        if (r2 <= 0.0) continue;
        loc[1]++;
        double q = sqrt(r2) * inv_h;
        if (q < 2.5) loc[2]++;
        if (q < 1.5) loc[3]++;
        if (q < 0.5) loc[4]++;
      }
    }
#pragma omp critical
    for (int k = 0; k < 5; ++k) tot[k] += loc[k];
  }
  free(act);
  for (int k = 0; k < 5; ++k) out5[k] = tot[k];
}
