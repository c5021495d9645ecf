// sph_kernels.h — internal launcher declarations shared by the host runtime (capi.cu).
#pragma once
#include "sph_common.cuh"

namespace sphb {

struct DenArgs;
struct ForArgs;
struct F2Args;

// pair sweeps (pair_kernels.cuh instantiations)
void launch_density_exact(const DenArgs &a, int n_items, bool aos, bool meanw, cudaStream_t s);
void launch_force_exact(const ForArgs &a, int n_items, bool aos, cudaStream_t s);
void launch_density_fast(const DenArgs &a, int n_items, bool aos, cudaStream_t s);
void launch_force_fast(const ForArgs &a, int n_items, bool aos, cudaStream_t s);
// issue-lean FAST force (builds its j-view first when n > 0); i side in the AoS records when
// F2Args::aos is set, else the SoA mirror; needs the per-stencil-cell periodic shift
// (nx, ny >= 5) and chunk boxes
void launch_force2(const F2Args &a, int n_items, int n, cudaStream_t s);
// split j-view for the issue-lean density round (density2_kernel, used by
// launch_density_fast when DenArgs::jv2.x is set)
struct D2View;
void launch_jview_density2(const D2View &v, const int *ilist, const Particle *aos,
                           const SoaMirror &f, bool use_aos, int n, cudaStream_t s);

// FAST j-views (kernels_fast.cu): sweep j fields in ilist order with hoisted invariants
void launch_jview_density(double2 *xy, double2 *vv, double *m, const int *ilist,
                          const Particle *aos, const SoaMirror &f, bool use_aos, int n,
                          cudaStream_t s);
void launch_jview_force(double2 *xy, double2 *vv, double2 *mg, double2 *pv, double *c,
                        const int *ilist, const Particle *aos, const SoaMirror &f, bool use_aos,
                        int n, double grav, cudaStream_t s);

// streaming kernels (kernels_exact.cu); kernel = SPH_DRIFT / SPH_KICK1 / SPH_KICK2
void launch_linear(int kernel, bool aos, Particle *p, const SoaMirror &f, int n, const Params &par,
                   cudaStream_t s);
void launch_eos(Particle *p, int n, double gamma, cudaStream_t s);
// exact counts of active pairs with q < 2.5, < 1.5, < 0.5 (reference arithmetic) into cnt[3]
void launch_pair_fractions(const Geom &g, const Item *items, int n_items, const int *list,
                           const SoaMirror &f, unsigned long long *cnt, cudaStream_t s);

// layout / bookkeeping kernels (kernels_layout.cu)
// AoS -> SoA for the fields in `mask` (the paper's gather view) and SoA -> AoS scatter.
void launch_gather(const Particle *aos, const SoaMirror &f, int n, uint32_t mask, cudaStream_t s);
void launch_scatter(Particle *aos, const SoaMirror &f, int n, uint32_t mask, cudaStream_t s);
// dense (host order) records -> device slots and back (full records)
void launch_expand(Particle *aos, const Particle *dense, const int *host_idx, int n, cudaStream_t s);
void launch_compact(Particle *dense, const Particle *aos, const int *host_idx, int n, cudaStream_t s);
// host-order records of slots [s0, s1) assembled from the resident SoA (+ AoS for the
// fields without a SoA array, at aos[home[slot]] when home is set)
void launch_compact_soa(Particle *dense, const Particle *aos, const SoaMirror &f,
                        const int *host_idx, const int *home, int s0, int s1, cudaStream_t s);
// domain decomposition: column-mask flags per slot, iota, indexed scatter
void launch_col_flags(unsigned char *flag, const Particle *aos, const SoaMirror &f, bool aos_src,
                      const unsigned char *mask, int n, int nx, int invert, cudaStream_t s);
void launch_iota(int *v, int n, cudaStream_t s);
void launch_scatter_idx(double *dst, const double *src, const int *idx, int m, cudaStream_t s);
// slot ranges of the pipelined force chunks; dep[g] = last chunk touching host chunk g
struct ChunkBounds {
  int k;      // chunks
  int s[33];  // slot bounds, s[0] = 0, s[k] = n (k <= 32)
};
void launch_host_chunk_dep(int *dep, const int *host_idx, int n, int hsz, const ChunkBounds &b,
                           cudaStream_t s);
// pack / unpack selected fields between device slots and a dense per-field buffer in host order.
// Buffer layout: for each field group in `mask` (ascending bit order) a block of n * size
// bytes, each block starting 16-byte aligned.
size_t packed_bytes(uint32_t mask, size_t n);
void launch_pack(char *dense, const Particle *aos, const int *host_idx, int n, uint32_t mask,
                 cudaStream_t s);
void launch_unpack_fields(Particle *aos, const char *dense, const int *host_idx, int n,
                          uint32_t mask, cudaStream_t s);
// spatial order of the locals within each cell (8x8 sub-cell bins); writes ilist
void launch_spatial_order(int *ilist, const Particle *aos, const SoaMirror &f, bool aos_src,
                          const int *cell_begin, int ncells, int nx, int ny, cudaStream_t s);
// work items from per-cell counts: items for cell c cover list[cell_begin[c] + k*kTI ...];
// out2[0] = n_items, out2[1] = pair count (sum cnt_c * na_c, int64 split in two ints)
// Items are emitted in `order` (cells sorted by descending cost bucket; may be null).
struct ItemsScratch {
  int *k, *off;     // ncells each
  void *tmp;        // cub scan temporary storage
  size_t tmp_bytes; // >= make_items_scratch_bytes(ncells)
};
size_t make_items_scratch_bytes(int ncells);
void launch_make_items(Item *items, int *n_items_out, long long *pairs_out, const int *cnt,
                       const int *cell_begin, const int *na_cell, const int *order, int ncells,
                       cudaStream_t s, int tile = 32, const ItemsScratch *scr = nullptr);
// FP32 bounding boxes of the 32-chunks of each cell's ilist (culled FAST density)
void launch_chunk_boxes(float4 *boxes, const int *ilist, const Particle *aos, const SoaMirror &f,
                        bool aos_src, const int *cell_begin, int ncells, cudaStream_t s);
// zero the work counts of cells that are not owned (domain decomposition halo)
void launch_mask_counts(int *cnt, unsigned *cost_key, const unsigned char *owned, int ncells,
                        cudaStream_t s);
// order-preserving per-cell compaction of the flagged (pending) list entries
void launch_compact_pending(int *out, int *cnt_out, const int *in, const int *cnt_in,
                            const unsigned char *again, const int *cell_begin, int ncells,
                            cudaStream_t s);
// per-cell active counts (sum of stencil cell counts) and per-cell local counts
// also writes a per-cell cost bucket key (8 per octave of nl*na) and order = identity
void launch_cell_counts(int *na_cell, int *cnt, unsigned *cost_key, int *order,
                        const int *cell_begin, int nx, int ny, cudaStream_t s);
// rebin helpers
void launch_rebin_keys(unsigned long long *keys, int *vals, int *cellnew, const Particle *aos,
                       const SoaMirror &f, bool aos_src, const long long *all_rank, int n, int nx,
                       int ny, cudaStream_t s);
void launch_cell_begin_from_sorted(int *cell_begin, const unsigned long long *keys, int n,
                                   int ncells, cudaStream_t s);
template <class T>
void launch_permute(T *dst, const T *src, const int *perm, int n, cudaStream_t s);
// record pieces of the fields without a SoA array only (id, cell, dbg[1], spare)
void launch_permute_record_tails(Particle *dst, const Particle *src, const int *perm, int n,
                                 cudaStream_t s);
void launch_set_cell(Particle *aos, const int *cell_begin, int ncells, cudaStream_t s);
// rebin by fix-up (capi.cu sph_ctx::rebin_fixup): movers only, merge order
struct FixupArgs {
  int n, ncells, nx, ny;
  const Particle *aos;
  SoaMirror soa;
  bool aos_src;
  const int *slot_cell, *cell_begin;
  const long long *all_rank;
  int *cellnew, *moved, *mpos, *out_cnt, *in_cnt, *in_begin, *in_fill, *inlist, *new_begin, *perm;
  void *scan_tmp;
  size_t scan_bytes;
};
size_t fixup_scan_bytes(int n);
void launch_rebin_fixup(const FixupArgs &a, cudaStream_t s);
// dst[k] = src[perm[k]] for the SoA mirror (soa), host_idx, all_rank, slot_cell := cellnew[perm]
// and, with rdst, the record tails (id, cell := new cell, dbg[1], spare)
// fused fix-up permute: slot k <- old slot perm[k] for the per-slot arrays (and the SoA
// mirror when `soa`); with home_dst set (resident mirror) the AoS record tails stay in place
// and home_dst[k] records where slot k's tail lives (home_src: the previous map, or null for
// identity), a mover's p->cell written there
void launch_permute_fused(const int *perm, int n, const SoaMirror &src, const SoaMirror &dst,
                          bool soa, const int *hid_src, int *hid_dst, const long long *ar_src,
                          long long *ar_dst, const int *cellnew, int *slot_cell,
                          const int *cell_old, const int *home_src, int *home_dst, Particle *aos,
                          bool step_dead, cudaStream_t s);
void launch_slot_cell_from_keys(int *slot_cell, const unsigned long long *keys, int n,
                                cudaStream_t s);
// device-resident decomposition: records of the selected slots from the SoA mirror + record
// tails (selection order); the 7-double halo payload (x, v_pred, m, p, c) out / in; the
// per-cell counts of a cell subset
void launch_export_soa(Particle *dense, const Particle *aos, const SoaMirror &f, const int *sel,
                       int m, cudaStream_t s);
void launch_export_halo(double *out, const SoaMirror &f, const int *sel, int m, cudaStream_t s);
void launch_append_halo(const SoaMirror &f_at, const double *in, int m, cudaStream_t s);
// density rounds >= 1: pending counts of the cells whose pending share is <= frac and count
// < dense_abs (sp, j-slice items) and of the others (dn, one lane per particle)
void launch_split_pending(int *sp, int *dn, const int *pend, const int *cnt, double frac,
                          int dense_abs, int ncells, cudaStream_t s);
void launch_subset_counts(int *out, const int *cnt, const unsigned char *mask, int ncells,
                          cudaStream_t s);
// FP64 DFMA throughput probe
void launch_fp64_probe(double *out, int blocks, int iters, cudaStream_t s);

} // namespace sphb
