// Host-side device execution plan (built once in kkt_dev_create; see plan.cpp).
#pragma once
#include <cstdint>
#include <vector>

#include "kkt_internal.h"

#define KKT_CTA_PHASE_MAX_ROWS 4096  // shared-memory rows of the single-CTA sweep phase

namespace kkt {

// Blocked sweep of the dense trailing block (sweep.cu): 32-column blocks in processing
// order.  Per block: the diagonal-triangle entries (CSR index -> tile position i*32+t) with a
// per-row presence mask, and the off-diagonal row segments (row, first CSR index, count)
// whose entries fall in the block's columns.
struct HostSweep {
  int32_t nblk = 0;
  int32_t max_stage = 0;  // largest number of off-diagonal entries of one block
  std::vector<int32_t> dptr, dsrc, bptr, brow, bbeg, bcnt, bofs;
  std::vector<uint16_t> ddst;
  std::vector<uint32_t> dmask;
};

struct HostPlan {
  int32_t n = 0;
  int64_t nnz_a = 0, in_nnz = 0, nnz_L = 0, nnz_U = 0;
  int has_lower = 0;
  // operator (general CSR) + value expansion + SpMV split points
  std::vector<int64_t> A_rp, A_ci, gen_src, A_split;
  // factors (CSC, position space) and permutations
  std::vector<int64_t> Lp, Up, row_perm, col_perm;
  std::vector<double> Lx0, Ux0, Udiag0;
  // refactor schedule
  std::vector<int64_t> so_ptr, ap_ptr;
  std::vector<int32_t> so_data, upd_ptr, a_src, col_order;
  std::vector<uint16_t> so_slot, upd_slot, a_slot;
  int32_t maxpat = 1, refactor_levels = 0;
  // leading levels refactorized thread-per-column: offsets into col_order (<= 8 levels)
  int32_t n_small_levels = 0;
  std::vector<int32_t> small_lev_ptr;
  // per so-entry metadata {slot of k in pattern(j), |L(:,k)|, first update pair, 0} and,
  // per update pair, the CSC index of the L(:,k) entry it consumes
  std::vector<int32_t> so_meta, upd_lidx;
  // trisolve CSR (L ascending cols, U descending cols) + CSC->CSR maps
  std::vector<int32_t> Lrp, Lci, Lmap, Urp, Uci, Umap;
  int32_t L_levels = 0, U_levels = 0;
  // trisolve phases.  L: rows [0, pL) grid-wide sync-free, rows [pL, n) one CTA (tail);
  // U: rows [pU, n) one CTA first (head), rows [0, pU) grid-wide.  Row orders by level.
  int32_t pL = 0, pU = 0, L_grid_levels = 0, U_grid_levels = 0;
  std::vector<int32_t> L_grid_order, L_tail_order, U_head_order, U_grid_order;
  // L_grid_order offsets of the leading levels run level-synchronously (L_sync_ptr.size()-1)
  std::vector<int32_t> L_sync_ptr;
  std::vector<int32_t> L_glev_ptr, U_glev_ptr;  // level boundaries in L/U_grid_order
  // per grid-order index: the row's critical (highest-level) grid dependency, or -1
  std::vector<int32_t> L_crit, U_crit;
  // per head column j >= pU: offset in U(:,j) (CSC, rows ascending) of the first row >= pU
  std::vector<int32_t> Uhead_off;
  std::vector<int32_t> Li32, Ui32;  // CSC row indices (int32) for the sweep phase
  std::vector<int32_t> Ltail_split;  // tail row r: CSR index of its first entry >= pL
  // U grid row r (< pU): CSR index of its first entry < pU (the head columns come first in the
  // descending CSR order); U_part_rows: the grid rows with at least one head entry
  std::vector<int32_t> Ugrid_split, U_part_rows;
  int32_t sweep_maxL = 0, sweep_maxU = 0;  // longest column inside each sweep block
  HostSweep swL, swU;
  // Single-system grid phases as chain tasks (build_chains): per task a code — row r (one
  // row), -(r+1) (external prefix of chain row r), or r0 | (m-1) << 26 (chain of m >= 2
  // rows from r0) — and an aux word (critical dependency, or the chain's partial-row mask);
  // per chain row the CSR index of its first internal entry.
  std::vector<int32_t> Lc_task, Lc_aux, Lc_split, Uc_task, Uc_aux, Uc_split;
};

// Tunables of the phase split (env KKT_TAIL_ROWS / KKT_HEAD_ROWS override the model).
int choose_tail(const HostPlan &P, bool upper);

int build_plan(const Symbolic &S, const int64_t *A_rp, const int64_t *A_ci, int64_t in_nnz,
               const int64_t *gen_src, HostPlan &P);

// Invariants of the chain task lists (kkt_plan_check).
void check_chains(const HostPlan &P, int64_t out[8]);

}  // namespace kkt
