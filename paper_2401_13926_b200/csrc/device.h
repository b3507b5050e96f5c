// Device handle + the launch interface between the host orchestration (device.cu, krylov.cu)
// and the kernel translation units (refactor.cu, trisolve.cu, vector.cu).
//
// A handle holds nb >= 1 same-pattern systems.  Every per-system array is system-major:
// system b's copy starts at b * (per-system size).  Kernels decompose their work into
// (task, system) pairs dispatched in dependency (level) order, so the dependency chains of
// all systems advance together in one launch (the batched path).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <vector>

#include "plan.h"

namespace kkt {

constexpr int RED_BLOCKS = 296;  // reduction blocks for one system (fixed => deterministic)
constexpr int RED_THREADS = 256;
constexpr double HAPPY_BREAKDOWN_RTOL = 1e-14;   // krylov.py:25
constexpr double PATCH_RELATIVE_FLOOR = 1e-12;   // direct_lu.py:32
constexpr int SCAL_STRIDE = 16;                  // per-system scalar block

// Blocked tail sweep tables (HostSweep, plan.h)
struct SweepDev {
  int nblk = 0, max_stage = 0;
  int *dptr = nullptr, *dsrc = nullptr, *bptr = nullptr, *brow = nullptr, *bbeg = nullptr,
      *bcnt = nullptr, *bofs = nullptr;
  uint16_t *ddst = nullptr;
  unsigned *dmask = nullptr;
};

// Device-side view of the plan + workspaces.  int32 indices on the device.
struct DevPlan {
  int n = 0, sym_lower = 0, has_lower = 0;
  int nb = 1;   // systems held
  // nb > 1: per-system arrays are INTERLEAVED [entry][nbp] (nbp = nb rounded up to 32; the
  // padding systems replicate system 0), so one warp serves 32 systems with coalesced
  // 256-byte accesses and SIMT-uniform control flow (batch.cu).  nb == 1: nbp == 1.
  int nbp = 1;
  int2 *btask = nullptr;  // batched refactor tasks {column, sys0 << 8 | log2(systems)}
  int n_btask = 0;
  int b_xbudget = 0, b_stage = 0, b_static = 0;
  int b_v2 = 0;  // light-column replay with two systems per lane (k_b_refactor2; KKT_B_V2)
  int b_xbudget2 = 0, b_stage2 = 0, n_btask1 = 0;  // second replay launch (wide columns)
  int ct_sc = 4;  // systems per k_b_refactor_cta task (KKT_B_CT_SC = 2 | 4 | 8)
  int ct_mode = 3;  // 3 (default): TMA pipeline; 0: entry x system lanes + CTA barrier per step;
                  // 1: warp per system; 2: 64 entry lanes (KKT_B_CT_MODE)
  // Heavy tail (columns >= J0, the dense separator; batched only): refactorized by a CTA per
  // (column, 32 systems) in "pull" form (k_b_refactor_heavy): every workspace slot sums its
  // own updates in the reference order, the slots spread over the CTA's warps, U slots
  // signal readiness through shared-memory flags.
  int J0 = 0x7fffffff;
  int nhc = 0, h_xp = 0;                   // heavy columns, their largest pattern
  int *hc_col = nullptr, *hc_optr = nullptr, *h_pp = nullptr;
  uint16_t *h_ord = nullptr;               // per heavy column: slots in pull order
  int2 *h_pairs = nullptr;                 // {source slot, L index}, slot-major, step order
  int *ticket2 = nullptr;
  // Wide columns through the TMA pipeline (k_b_refactor_tma, ct_mode 3): a producer warp
  // stages each chunk's L(:,k) rows (2-D tensor maps over Lx viewed as [nnz_L][nbp], boxes of
  // 128 / 32 / 8 rows x 8 systems) and update slots (1-D bulk copies) into an mbarrier ring
  // once the dependency column's done flag is up; the consumer warps only replay.
  int J2 = 0x7fffffff;                     // first wide column
  int so_dep0 = 0;                         // so index of the first wide column's first step
  int *so_dep = nullptr;                   // per wide-column step: k - J2 (wide k) or -1
  int *cflag = nullptr;                    // [(j - J2) * nbp / 8 + group]: L(:,j) published
  int tma_ns = 2, tma_stg = 256;           // stages x rows (KKT_B_TMA)
  int tma_e = 32;                          // entry lanes per system (64: one CTA per SM; KKT_B_TMA_E)
  int tma_direct = 2;                      // late steps: 2 value-as-flag L2 reads (KKT_B_TMA_DIRECT)
  CUtensorMap tmL[3];                      // Lx boxes of 128, 32, 8 rows x 8 systems
  unsigned long long *prof = nullptr;  // optional per-warp cycle counters (KKT_TRACE, batched)
  int rb = RED_BLOCKS;  // reduction blocks per system
  int64_t nnz_a = 0, in_nnz = 0, in_cap = 0, nnz_L = 0, nnz_U = 0, n_so = 0, n_upd = 0, n_ap = 0;
  int maxpat = 1;
  int ref_start = 0;       // first col_order index handled by the warp kernel
  int n_small_levels = 0;  // leading levels run by k_refactor_small
  int lev_ptr[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};  // col_order offsets of those levels
  int poll_ns = 0;  // __nanosleep back-off while polling (env KKT_POLL_NS)
  int ref_buf = 256;  // single-system refactor: update pairs per stage buffer (two buffers)
  int ref_direct = 1;  // single-system refactor: lanes poll their own unpublished L entries
  // single-system refactor: col_order[ref_start, ref_start + ref_n1) = the columns of the warp
  // kernel (k_refactor), the rest (j >= JW, reordered after them, level order kept) the wide
  // columns of k_refactor_wide (KKT_REF_WIDE_NP; ring slot / staged steps / launch shape)
  int ref_n1 = 0, ref_wslot = 0, ref_wsteps = 0, ref_wblocks = 0, ref_wnt = 256;
  size_t ref_wsmem = 0;
  int grid_wait = 0;  // sync-free grid solves: 1 = wait on a row's critical dependency first
  // operator (pattern shared; values per system)
  int *A_rp, *A_ci, *A_split, *gen_src;
  double *in_vals, *A_vals;                 // [nb][in_cap], [nb][nnz_a]
  double *in_il = nullptr;                  // batched: caller values interleaved [in_cap][nbp]
  // refactor (schedule shared)
  int *so_ptr, *ap_ptr, *a_src, *col_order, *Lp, *Up, *Lmap, *Umap, *upd_lidx;
  int4 *so_meta;
  uint16_t *upd_slot, *a_slot;
  int *upd_slot32 = nullptr;               // batched: int32 slots (in the upd_lidx buffer)
  double *Lx, *Ux, *udiag;                  // [nb][nnz_L], [nb][nnz_U], [nb][n]
  // trisolves (pattern/schedule shared)
  int *Lrp, *Lci, *Urp, *Uci, *row_perm, *col_perm;
  int *L_grid_order, *L_tail_order, *U_head_order, *U_grid_order;
  int *L_crit, *U_crit, *Uhead_off, *Li, *Ui, *Ltail_split;
  int *Ugrid_split = nullptr, *U_part_rows = nullptr;  // U grid rows' head prefix (plan.h)
  int n_upart = 0, u_partial = 1;  // rows with a head prefix; 0 = grid rows sum it (KKT_U_PARTIAL)
  double *tacc;                             // [nb][n - pL] tail partial sums (grid -> sweep)
  int pL, pU, nLg, nUg;                     // split positions and grid-phase row counts
  // single-system chain tasks of the grid phases (plan.h build_chains; KKT_CHAINS=0: off)
  int *Lc_task = nullptr, *Lc_aux = nullptr, *Lc_split = nullptr;
  int *Uc_task = nullptr, *Uc_aux = nullptr, *Uc_split = nullptr;
  int nLc = 0, nUc = 0, chains = 0;
  double *cpart = nullptr;                  // [n] chain rows' external prefix (sentinel-reset)
  int L_nsync = 0, L_sync_ptr[5] = {0, 0, 0, 0, 0};  // level-synchronous leading L levels
  int *L_glev = nullptr, *U_glev = nullptr;  // level boundaries of the grid orders
  int L_nglev = 0, U_nglev = 0;
  unsigned *gbar = nullptr;                   // grid barrier {count, generation}
  int b_levelsync = 0;  // batched grid phases level-synchronous (KKT_B_LEVELSYNC=1; slower here)
  int b_gridv = 3;      // batched grid-solve variant the persistent grid was sized for
  int sweep_maxL, sweep_maxU;
  SweepDev swL, swU;                        // blocked sweeps of the trailing blocks
  double *Lv, *Uv;                          // [nb][nnz_L], [nb][nnz_U] (CSR order)
  double *yL, *yU;                          // [nb][n] sentinel-reset (value == readiness)
  // optional timeline (KKT_TRACE=1), system 0 only
  unsigned long long *trace_ref, *trace_trsv, *trace_step;
  // scalars
  unsigned long long *scal;                 // [nb][SCAL_STRIDE]
  int *ticket;
  double *partials;                         // [nb][8][rb]
  // systems to process (nullptr = all).  A system may skip a whole solve: after a complete
  // solve yL is all-sentinel and yU published, which is exactly the state a solve expects.
  const int *sys_mask = nullptr;
};

// 32-bit index arithmetic: kkt_dev_create rejects batches whose interleaved arrays exceed
// 2^32 elements, so the product never wraps.
__host__ __device__ __forceinline__ size_t IL(const DevPlan &d, int64_t i, int sys) {
  return (size_t)((unsigned)i * (unsigned)d.nbp + (unsigned)sys);
}

__device__ __forceinline__ bool sys_active(const DevPlan &d, int sys) {
  return d.sys_mask == nullptr || d.sys_mask[sys] != 0;
}

// indices into a system's scalar block (bit patterns of non-negative doubles unless noted)
enum {
  SC_MAXABS_A = 0,  // max |a|
  SC_INFNORM,       // ||A||_inf of the general matrix (row sums in entry order)
  SC_GMAX,          // growth numerator (refactorize)
  SC_PATCHED,       // integer count
  SC_MAXPIV,        // max |u_jj|
  SC_MINPIV,        // min |u_jj|
  SC_NONFINITE,     // integer flag
  SC_OPNORM,        // ||K||_inf of the operator as the reference computes it
  SC_COUNT
};

struct Krylov;  // FGMRES workspace (krylov.cu)

struct Device {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t stream2 = nullptr;          // batched: the wide-column replay, run alongside
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  DevPlan d;
  HostPlan h;
  void *arena = nullptr;
  void *trace_mem = nullptr;
  size_t arena_bytes = 0;
  int sm_count = 0;
  int refactor_blocks = 0, refactor_warps = 8, refactor_blocks2 = 0, refactor_blocks_ov = 0;
  size_t refactor_smem2 = 0;
  size_t refactor_smem = 0;
  int trsv_blocks = 0;
  int trsv_blocks_full = 0;  // the grid solve's full-GPU persistent grid (helpers may use less)
  long long launches = 0;
  Krylov *kry = nullptr;
  double *pinned = nullptr;  // pinned host staging (status words)
  size_t pinned_bytes = 0;
  int restart_m = 10;
  // Straggler helpers (batched handles): single-system handles over the same plan that take
  // over the FGMRES of the last few running systems of a batch (krylov.cu, handoff).
  std::vector<Device *> helpers;
  cudaEvent_t ev_h = nullptr;
};

// a handle of width `batch` over src's host plan (device.cu)
int create_like(const Device *src, int batch, Device *&out);

// ---- launchers (each returns cudaGetLastError of its launch) ----
cudaError_t launch_expand_norms(const DevPlan &d, cudaStream_t s);
cudaError_t launch_reset_scal(const DevPlan &d, int mode, cudaStream_t s);
cudaError_t launch_refactor(const DevPlan &d, int blocks, int warps, size_t smem, cudaStream_t s,
                            long long *launches);
cudaError_t launch_diag_stats(const DevPlan &d, int blocks, cudaStream_t s);
cudaError_t refactor_configure(int warps, size_t smem, int buf, int *blocks_per_sm);
size_t refactor_smem_bytes(int warps, int maxpat, int buf);
size_t refactor_wide_smem(int maxpat, int maxsteps, int slot);
cudaError_t refactor_wide_configure(int nt, size_t smem, int *blocks_per_sm);
int refactor_wide_nt(double mean_step);  // CTA width of k_refactor_wide (KKT_REF_WIDE_NT)
int refactor_buf();  // KKT_REF_BUF (refactor.cu)

cudaError_t launch_trsv(const DevPlan &d, const double *b, double *x, int grid_blocks,
                        cudaStream_t s, long long *launches);
cudaError_t trsv_configure(int *grid_blocks_per_sm);
// L phase up to the sweep (row-parallel leading levels, sync-free grid, tail partial sums)
cudaError_t launch_L_front(const DevPlan &d, const double *b, double *x, int grid_blocks, cudaStream_t s,
                           long long *launches);
cudaError_t b_launch_grid_L(const DevPlan &d, const double *b, double *x, int grid_blocks, cudaStream_t s);
cudaError_t launch_fill_sentinel(double *p, int64_t n, cudaStream_t s);
cudaError_t launch_add_inplace(double *x, const double *y, int64_t n, cudaStream_t s);
// the U grid rows' head-column prefix sums into yL (row-parallel; after the U sweep)
cudaError_t launch_U_partial(const DevPlan &d, cudaStream_t s, long long *launches);
// blocked sweep of the trailing block (sweep.cu), single and batched handles
cudaError_t sweep_configure();
cudaError_t launch_sweep_blocked(const DevPlan &d, bool upper, double *x, cudaStream_t s);

// ---- batched (interleaved, nb > 1) kernels: batch.cu ----
constexpr int B_XBUDGET = 576;   // default refactor workspace doubles per warp (np * systems)
constexpr int B_STAGE = 256;     // default stage buffer doubles (pairs * systems), x2 buffers
constexpr int B_XBUDGET2 = 2304;  // ... for the wide separator columns (second launch)
constexpr int B_STAGE2 = 768;
constexpr int B_WARPS = 4;       // warps per refactor CTA
size_t b_refactor_smem(int xbudget, int stage);
int b_grid_variant();  // KKT_B_GRIDV (batch.cu)
cudaError_t b_configure(int nbp, size_t refactor_smem, int gridv, int *refactor_blocks_per_sm,
                        int *trsv_blocks_per_sm);
cudaError_t b_launch_expand_norms(const DevPlan &d, cudaStream_t s);
cudaError_t b_launch_refactor(const DevPlan &d, int blocks, size_t smem, int blocks2, size_t smem2,
                              cudaStream_t s, long long *launches, cudaStream_t s2 = nullptr,
                              cudaEvent_t ev_a = nullptr, cudaEvent_t ev_b = nullptr, int blocks_ov = 0);
cudaError_t b_refactor_occupancy(size_t smem, int *blocks_per_sm);
size_t b_cta_smem(int xp, int sc);
void b_tma_shape(int xp, int *ns, int *stg);
size_t b_tma_smem(int xp, int ns, int stg);
cudaError_t b_tma_configure(int ns, int stg, int e, bool flags, size_t smem, int *blocks_per_sm);
cudaError_t b_tma_maps(DevPlan &d);  // encode d.tmL over d.Lx
cudaError_t b_cta_configure(int sc, size_t smem, int *blocks_per_sm, bool wide);
cudaError_t b_launch_diag_stats(const DevPlan &d, cudaStream_t s);
cudaError_t b_launch_trsv(const DevPlan &d, const double *b, double *x, int grid_blocks,
                          cudaStream_t s, long long *launches);
cudaError_t b_launch_spmv(const DevPlan &d, const double *x, double *out, const double *bsub,
                          double *nrm_partials, cudaStream_t s);
cudaError_t b_launch_resid_stats(const DevPlan &d, const double *r, const double *x,
                                 double *partials, double *out5, cudaStream_t s);
// [nb][n] (system-major, caller layout) <-> [n][nbp] (interleaved); padding <- system 0
cudaError_t b_launch_to_il(const DevPlan &d, const double *src, double *dst, cudaStream_t s);
cudaError_t b_launch_from_il(const DevPlan &d, const double *src, double *dst, cudaStream_t s);
cudaError_t b_launch_transpose(const DevPlan &d, const double *src, int64_t count, double *dst,
                               cudaStream_t s);  // [nb][count] -> [count][nbp]
cudaError_t b_launch_broadcast(const double *src, int64_t count, int nbp, double *dst, cudaStream_t s);
constexpr int B_HEAVY_SMEM_MAX = 200 * 1024;  // dynamic shared memory of k_b_refactor_heavy
size_t b_heavy_smem(int xp);
// FGMRES vector kernels on interleaved [n][nbp] vectors (partials [nbp][nvec][rb])
cudaError_t b_launch_dots(const DevPlan &d, const double *V, int nvec, const double *w,
                          const int *mask, double *partials, cudaStream_t s);
cudaError_t b_launch_cgs(const DevPlan &d, const double *V, int nvec, const double *w_in,
                         const double *h, int hstride, double *w_out, int mode, const int *mask,
                         double *partials, cudaStream_t s);
cudaError_t b_launch_cgs_dots(const DevPlan &d, const double *V, int nvec, const double *w_in,
                              const double *h, int hstride, double *w_out, const int *mask,
                              double *partials, cudaStream_t s);  // nvec <= 16
cudaError_t b_launch_scale(const DevPlan &d, const double *in, double *out, const double *den,
                           int dstride, const int *mask, cudaStream_t s);
cudaError_t b_launch_update_x(const DevPlan &d, double *x, const double *Z, const double *y,
                              int ystride, const int *jused, cudaStream_t s);

// vectors are [nb][n]; partials are [nb][nvec][rb]; out is [nb][nvec]
cudaError_t launch_spmv(const DevPlan &d, const double *x, double *out, const double *bsub,
                        double *nrm_partials, cudaStream_t s);
cudaError_t launch_reduce_partials(const DevPlan &d, const double *partials, int nvec, double *out,
                                   int ostride, int op_sqrt, cudaStream_t s);
cudaError_t launch_resid_stats(const DevPlan &d, const double *r, const double *x,
                               double *partials, double *out5, cudaStream_t s);

}  // namespace kkt
