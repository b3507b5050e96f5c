// Device handle: every buffer the hot path needs, allocated once (one arena).
#pragma once
#include <cuda_runtime.h>

#include "plan.h"

namespace kkt {

// Device-side view of the plan + workspaces.  int32 indices everywhere on the device.
struct DevPlan {
  int n = 0, sym_lower = 0, has_lower = 0;
  int64_t nnz_a = 0, in_nnz = 0, nnz_L = 0, nnz_U = 0, n_so = 0, n_upd = 0, n_ap = 0;
  int maxpat = 1;
  // operator
  int *A_rp, *A_ci, *A_split, *gen_src;
  double *in_vals, *A_vals;
  // refactor
  int *so_ptr, *so_data, *upd_ptr, *ap_ptr, *a_src, *col_order, *Lp, *Up, *Lmap, *Umap;
  uint16_t *so_slot, *upd_slot, *a_slot;
  double *Lx, *Ux, *udiag;
  int *done;
  // trisolves
  int *Lrp, *Lci, *Urp, *Uci, *L_order, *U_order, *row_perm, *col_perm;
  double *Lv, *Uv;
  int *tflag;
  double *y;
  // scalar block (device): see Scal
  unsigned long long *scal;
  int *ticket;
  double *partials;
};

// indices into DevPlan::scal (bit patterns of non-negative doubles unless noted)
enum {
  SC_MAXABS_A = 0,    // max |a|
  SC_INFNORM,         // ||A||_inf  (row sums in entry order)
  SC_GMAX,            // growth numerator (refactorize)
  SC_PATCHED,         // integer count
  SC_MAXPIV,          // max |u_jj|
  SC_MINPIV,          // min |u_jj|
  SC_NONFINITE,       // integer flag
  SC_COUNT
};

struct Krylov;  // FGMRES workspace (device.cu)

struct Device {
  int device = 0;
  cudaStream_t stream = nullptr;
  DevPlan d;
  HostPlan h;
  void *arena = nullptr;
  size_t arena_bytes = 0;
  int sm_count = 0;
  int refactor_blocks = 0, refactor_warps = 8;
  size_t refactor_smem = 0;
  int trsv_blocks = 0;
  int epoch_refactor = 0, epoch_trsv = 0;
  long long launches = 0;
  Krylov *kry = nullptr;
  double *pinned = nullptr;  // small pinned host staging buffer
  int restart_m = 10;
};

}  // namespace kkt
