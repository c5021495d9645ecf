/* sph_b200.h — C-ABI drop-in for the reference SPH hot path on B200 (sm_100a).
 *
 * The reference's boundary is
 *   KernelTimes soaview::sph::run_sweep(KernelId k, const CellGrid &grid,
 *                                       const SphParams &par, Path path, Order order,
 *                                       Guard guard, int threads = 1);
 *   (/root/reference/proj/include/soaview/sph/kernels.hpp:45-46, kernels.cpp:861-872)
 * which mutates the caller's 272-byte AoS `Particle` records (particle.hpp:11-46) in place
 * through the per-cell `local` / `active` pointer lists of a `CellGrid` (grid.hpp:32-40).
 *
 * This header exposes the same operation as plain C: the caller flattens
 * CellGrid::local into one `Particle*` array (cell-major) plus `cell_begin[ncells+1]`;
 * the active lists are the reference's deduplicated, wrapped 3x3 stencil
 * (grid.cpp:159-182) and are implied by (nx, ny). The library keeps a device-resident
 * mirror of the records; sweeps run entirely on the GPU; sph_download writes back only
 * the bytes the kernels wrote (each kernel's A_out, kernels.cpp:741-859, plus `flags`).
 *
 * Conventions: every function returns 0 on success and a negative SPH_E* code on error
 * (details via sph_last_error). No C++ exceptions cross this boundary. Calls on one
 * context are serialised by the caller; host pointers are borrowed for the call only.
 * Integer selector values equal the reference enums (KernelId, Path, Order, Guard).
 */
#ifndef SPH_B200_H
#define SPH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPH_B200_ABI_VERSION 1
#define SPH_RECORD_SIZE 272 /* sizeof(soaview::sph::Particle), particle.hpp:40 */

/* error codes */
#define SPH_OK 0
#define SPH_E_ARG -1     /* invalid argument */
#define SPH_E_CUDA -2    /* CUDA runtime error (no device, OOM, launch failure) */
#define SPH_E_STATE -3   /* call out of order (e.g. sweep before bind) */

/* KernelId, kernels.hpp:9 */
enum { SPH_DENSITY = 0, SPH_FORCE = 1, SPH_DRIFT = 2, SPH_KICK1 = 3, SPH_KICK2 = 4 };
/* Path, kernels.hpp:13 */
enum { SPH_PATH_AOS_BASELINE = 0, SPH_PATH_SOA_VIEW = 1 };
/* Order, kernels.hpp:17 */
enum { SPH_ORDER_LOCAL_ACTIVE = 0, SPH_ORDER_ACTIVE_LOCAL = 1 };
/* Guard, kernels.hpp:20 */
enum { SPH_GUARD_BRANCH = 0, SPH_GUARD_MASK = 1 };
/* Device layout mode (the layout ablation). FROM_PATH maps AosBaseline -> AOS and
 * SoaView -> CONVERT, mirroring the reference's two access paths. */
enum { SPH_LAYOUT_FROM_PATH = -1, SPH_LAYOUT_AOS = 0, SPH_LAYOUT_CONVERT = 1,
       SPH_LAYOUT_RESIDENT = 2 };
/* Numerics. EXACT reproduces the reference's floating-point operation sequence (no FMA,
 * IEEE sqrt/div, reference j order) and is byte-identical to the CPU. FAST uses FMA,
 * rsqrt+Newton and hoisted per-j terms; results agree within the documented tolerance. */
enum { SPH_NUMERICS_EXACT = 0, SPH_NUMERICS_FAST = 1 };

typedef struct sph_ctx sph_ctx;

/* SphParams, particle.hpp:49-55 (same field order). */
typedef struct {
  double dt, gamma, cfl, grav, target_wcount;
} sph_params;

/* KernelTimes, kernels.hpp:24-29 (device-measured: prologue = H2D/AoS->SoA,
 * compute = kernels, epilogue = SoA->AoS/D2H). */
typedef struct {
  int64_t prologue_ns, compute_ns, epilogue_ns;
} sph_times;

typedef struct {
  int64_t n;                  /* bound particles */
  int32_t nx, ny, ncells;
  int32_t layout, numerics;
  int64_t active_pairs;       /* sum over cells of nl*na (one pass) */
  int64_t density_pairs;      /* last density sweep: sum of nl*na*rounds */
  int64_t density_updates;    /* last density sweep: particle-rounds */
  int32_t density_rounds;     /* last density sweep: max rounds */
  int32_t pad0;
  int64_t density_failures;   /* last density sweep: particles that hit 30 rounds */
  int64_t force_pairs;        /* last force sweep: sum of nl*na */
  double last_density_ms, last_force_ms; /* device time of the pair kernels */
  double density_round_ms[4];   /* last density sweep: kernel time of rounds 1-4 */
} sph_stats;

int sph_abi_version(void);

/* Context lifetime (one per device; owns a CUDA stream). */
int sph_create(int device, sph_ctx **out);
void sph_destroy(sph_ctx *ctx);
const char *sph_last_error(const sph_ctx *ctx);

int sph_set_numerics(sph_ctx *ctx, int numerics);
int sph_set_layout(sph_ctx *ctx, int layout);

/* Bind a CellGrid. recs[k] for k in [cell_begin[c], cell_begin[c+1]) are the records of
 * CellGrid::local[c] in list order; ncells = nx*ny. all_rank (optional, may be NULL) gives
 * each record's index in ParticleStore::all, used to reproduce build_grid's list order on
 * device rebins (grid.cpp:152-158); NULL means the flattened order itself. Uploads every
 * record (all 272 bytes) to the device mirror. */
int sph_bind(sph_ctx *ctx, void *const *recs, const int64_t *cell_begin, int nx, int ny,
             double cell_size, const int64_t *all_rank);

/* Domain decomposition: sweeps compute only the cells with owned[c] != 0 (NULL = all);
 * particles of other bound cells (halo) still appear in the active lists but are not
 * updated by density / force. Takes effect immediately and survives rebins. */
int sph_set_owned_cells(sph_ctx *ctx, const uint8_t *owned);

/* Re-upload all records (host mutated them); recs in the bound order. */
int sph_upload(sph_ctx *ctx, void *const *recs);

/* Write back the fields written on the device since the last upload/download (the A_out
 * of each kernel run, plus flags); all other bytes of the host records stay untouched.
 * recs are in the bound order (the device tracks rebins internally). */
int sph_download(sph_ctx *ctx, void *const *recs);

/* Write back every byte of every record. */
int sph_download_all(sph_ctx *ctx, void *const *recs);

/* One sweep of kernel `kernel` on the device mirror (no host traffic). */
int sph_sweep(sph_ctx *ctx, int kernel, const sph_params *par, int path, int order, int guard,
              sph_times *times);

/* Drop-in for run_sweep on host records: upload (if the context is not already in sync),
 * sweep, download of the kernel's A_out. times: prologue = H2D, epilogue = D2H. */
int sph_run_sweep(sph_ctx *ctx, int kernel, void *const *recs, const sph_params *par,
                  int path, int order, int guard, sph_times *times);

/* One leapfrog step on HOST records (the end-to-end drop-in): every record of the bound
 * order is copied host->device, the step runs on the device (kick1 -> drift -> rebin ->
 * density -> force -> kick2), and every record is copied back. recs in the bound order.
 * kernel_ms (optional, 8 entries): H2D, the six phases, D2H (device time). */
int sph_step_host(sph_ctx *ctx, void *const *recs, const sph_params *par, double *kernel_ms);

/* drift_one / kick1_one / kick2_one (kernels.hpp:52-54, kernels.cpp:880-893) on n dense host
 * records (272 B each, in place): copied to a device scratch buffer, updated by the exact
 * streaming kernel, copied back. Independent of the bound grid. kernel: SPH_DRIFT, SPH_KICK1
 * or SPH_KICK2. */
int sph_apply_records(sph_ctx *ctx, int kernel, void *records, int64_t n, const sph_params *par);

/* Page-lock a host range for full-bandwidth copies (cudaHostRegister); optional. */
int sph_host_register(sph_ctx *ctx, void *base, uint64_t bytes);
int sph_host_unregister(sph_ctx *ctx, void *base);

/* Rebuild the cell lists on the device after particles moved (build_grid,
 * grid.cpp:145-184): cell = clamp(floor(x*nx)), list order by ParticleStore::all rank. */
int sph_rebin(sph_ctx *ctx);

/* One leapfrog step on the device: kick1 -> drift -> rebin -> density -> force -> kick2.
 * kernel_ms (optional, 6 entries) receives per-phase device time in that order. */
int sph_step(sph_ctx *ctx, const sph_params *par, double *kernel_ms);

/* make_particles (grid.cpp:76-143) on the device: the reference's deterministic IC
 * (mt19937_64 on the host, then grid, mean_wcount, density, EOS and force with EXACT
 * numerics, so records are byte-identical to the reference's) bound as a continuous
 * store (ParticleStore::all sorted by (cell, id)). par_out receives the calibrated params. */
int sph_make_particles(sph_ctx *ctx, int64_t n, int ppc, uint64_t seed, sph_params *par_out);

/* Initial-condition kinds for sph_make_particles_ex. UNIFORM is the reference's
 * make_particles. CLUSTERED is the builder-defined variable-ppc IC of BASELINE config 3
 * (the reference has none): the same RNG stream and pipeline, but half of the particles
 * sit in 16 Gaussian clumps (sigma = 1 cell, centres drawn first, Irwin-Hall(12)
 * deviates, wrapped with x - floor(x)); restated identically in oracle/sph_oracle.c. */
enum { SPH_IC_UNIFORM = 0, SPH_IC_CLUSTERED = 1 };
int sph_make_particles_ex(sph_ctx *ctx, int64_t n, int ppc, uint64_t seed, int kind,
                          sph_params *par_out);

/* Copy the mirror into a dense host array of n records in bound order (ParticleStore::all
 * order for sph_make_particles contexts). */
int sph_read_records(sph_ctx *ctx, void *out_records);

/* Counters and timings of the last sweeps / step. Counts that are still in flight to the host
 * (the work list built by the last rebin) are waited for, so this may synchronise the
 * context's stream. */
int sph_get_stats(const sph_ctx *ctx, sph_stats *out);
int sph_synchronize(sph_ctx *ctx);

/* Measured FP64 FMA throughput of this device (TFLOP/s, 2 flops per DFMA). */
int sph_fp64_peak(sph_ctx *ctx, double *tflops);

/* Exact support fractions of the current state, a validation pass outside any timed
 * region: out[0..2] = the shares of all active pairs (sum over cells of
 * nl * na, out[3]) with q < 2.5, q < 1.5, q < 0.5, q = |x_i - x_j| / h_i by the reference's
 * arithmetic (kernels.cpp:97-108). They fix the algorithmic flops per pair of bench.py. */
int sph_pair_fractions(sph_ctx *ctx, double out[4]);

/* ---- Device-resident slab decomposition (paper_2502_16517_b200/decomp.py) ----
 * The reference has no decomposition; these entry points let one context per GPU hold its
 * slab's particles on the device while the halo / migration traffic moves between GPUs as
 * device buffers (NCCL). col_mask is a HOST array of nx bytes selecting cell columns; a
 * particle's column is build_grid's clamp(floor(x * nx)) (grid.cpp:153) of its current x.
 * Record / rank / rho buffers are DEVICE pointers. All calls synchronise the context.
 *   sph_dd_count       particles in the selected columns
 *   sph_dd_export      copy their records (272 B, current values) and all-ranks out, in slot
 *                      order (after sph_rebin: (cell, all-rank) order)
 *   sph_dd_remove      drop them (the remaining slots keep their order)
 *   sph_dd_append      add m records (+ all-ranks); pair sweeps then need sph_rebin
 *   sph_dd_export_rho / sph_dd_import_rho
 *                      rho of the selected particles out / in, in slot order (the halo
 *                      refresh between density and force: force reads the active
 *                      particles' rho, kernels.cpp:443-456)
 * Host-order views (sph_read_records) of a context changed by these calls are in slot
 * order. */
int sph_dd_count(sph_ctx *ctx, const uint8_t *col_mask, int64_t *count);
int sph_dd_export(sph_ctx *ctx, const uint8_t *col_mask, void *dev_recs, int64_t *dev_ranks,
                  int64_t cap, int64_t *count);
int sph_dd_remove(sph_ctx *ctx, const uint8_t *col_mask);
int sph_dd_append(sph_ctx *ctx, const void *dev_recs, const int64_t *dev_ranks, int64_t m);
int sph_dd_export_rho(sph_ctx *ctx, const uint8_t *col_mask, double *dev_out, int64_t cap,
                      int64_t *count);
int sph_dd_import_rho(sph_ctx *ctx, const uint8_t *col_mask, const double *dev_in, int64_t m);
/* Halo records as the pair sweeps read them from an active particle that is not a local of
 * an owned cell: x[2], v_pred[2], m, p, c (7 doubles = 56 B per particle, kernels.cpp:379-456
 * ActiveView fields minus rho, which follows after density through sph_dd_export_rho) plus
 * the all-rank. sph_dd_append_halo adds such particles (every other field zero); they must
 * stay outside the owned cells and be dropped (sph_dd_remove) after the step. */
int sph_dd_export_halo(sph_ctx *ctx, const uint8_t *col_mask, double *dev_out, int64_t *dev_ranks,
                       int64_t cap, int64_t *count);
int sph_dd_append_halo(sph_ctx *ctx, const double *dev_in, const int64_t *dev_ranks, int64_t m);
/* The force sweep on the owned cells c with cell_mask[c] != 0 (HOST array of ncells bytes):
 * a decomposed step runs the halo-independent interior while the halo rho is in flight. */
int sph_sweep_cells(sph_ctx *ctx, int kernel, const sph_params *par, const uint8_t *cell_mask);
/* Run the context's device work on `stream` (a cudaStream_t; NULL: the context's own), e.g.
 * the caller's NCCL-ordered stream. */
int sph_set_stream(sph_ctx *ctx, void *stream);
/* Local particle count of every cell (ncells int64 values, HOST array). */
int sph_cell_counts(sph_ctx *ctx, int64_t *out);
/* Current particle count of the context. */
int64_t sph_count(const sph_ctx *ctx);

/* Number of kernel launches issued by this library so far (for bench accounting). */
int64_t sph_launch_count(const sph_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* SPH_B200_H */
