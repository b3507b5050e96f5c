// Triangular solves x = lu_solve(b) (direct_lu.py:359-379), bitwise with the reference.
//
// The reference sweeps columns: forward `y[Li(j)] -= Lx(j)*y[j]` for ascending j, backward
// `y_j /= u_jj; y[Ui(j)] -= Ux(j)*y_j` for descending j.  Row r therefore receives its
// updates in ascending column order (L) / descending column order (U).  Both schedules below
// preserve that per-row order, with separately rounded products, so every bit matches.
//
// Per sweep the rows split at a position chosen on the host from the level profile
// (plan.cpp choose_tail):
//   * grid phase (wide part of the DAG) — persistent, sync-free, warp per row, rows
//     round-robin in level order.  Readiness is the value itself: y is reset to a sentinel
//     NaN pattern and consumers re-read y[col] until it is published.  Only ONE lane polls,
//     on the row's critical (highest-level) dependency, so a just-published value is not
//     hammered by every row of a dense separator (that L2 hot spot cost ~10 us per hop);
//   * sweep phase (the dense separator at the end of the elimination order) — one CTA
//     sweeps the block 32 columns at a time (sweep.cu: a shuffle chain for the diagonal
//     triangle, row-parallel updates below it), keeping the reference's per-row order.
//   L = [grid rows < pL] then [sweep columns pL..n-1];
//   U = [sweep columns n-1..pU] then [grid rows < pU].
// Each sweep resets the other sweep's buffer for the next solve, so no memsets are needed.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "device.h"
#include "kernels.cuh"

namespace kkt {




// ---- grid phase: warp per row ------------------------------------------------------------
template <bool IS_U>
__global__ void __launch_bounds__(256) k_trsv_grid(DevPlan d, const double *__restrict__ b,
                                                   double *__restrict__ xout) {
  const int lane = threadIdx.x & 31;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int *order = IS_U ? d.U_grid_order : d.L_grid_order;
  const int *crit = IS_U ? d.U_crit : d.L_crit;
  const int nrows = IS_U ? d.nUg : d.nLg;
  const int *rp = IS_U ? d.Urp : d.Lrp;
  const int *ci = IS_U ? d.Uci : d.Lci;
  const int64_t nnz = IS_U ? d.nnz_U : d.nnz_L;
  const int ntask = nrows * d.nb;
  const int gstart = IS_U ? 0 : d.L_sync_ptr[d.L_nsync];  // leading levels ran row-parallel
  // task = (level-ordered row index, system): row-major so all systems' copies of a row
  // are adjacent and every dependency of a task has a smaller task index
  for (int task = gstart * d.nb + gwarp; task < ntask; task += nwarps) {
    const int idx = task / d.nb, sys = task % d.nb;
    if (!sys_active(d, sys)) continue;
    const int r = order[idx];
    const double *vals = (IS_U ? d.Uv : d.Lv) + (size_t)sys * nnz;
    double *ysrc = (IS_U ? d.yU : d.yL) + (size_t)sys * d.n;  // published by this sweep
    double *yres = (IS_U ? d.yL : d.yU) + (size_t)sys * d.n;  // reset for the next solve
    const int beg = (IS_U && d.u_partial) ? d.Ugrid_split[r] : rp[r], end = rp[r + 1];
    // independent loads first: the initial value and the first chunk's pattern/values
    double acc = IS_U ? ldcg(&d.yL[(size_t)sys * d.n + r]) : b[(size_t)sys * d.n + d.row_perm[r]];
    const double piv = IS_U ? d.udiag[(size_t)sys * d.n + r] : 1.0;  // off the critical path
    int col = 0;
    double v = 0.0;
    if (beg + lane < end) {
      col = ci[beg + lane];
      v = vals[beg + lane];
    }
    // grid_wait 1 (the single-system default): lane 0 alone spins on the critical dependency
    // before the row; the other dependencies are then normally published already, so the
    // lanes' loads below rarely have to wait.  (0: each lane polls its own unpublished column
    // in the chunk loop — many pollers per row, measured 2.5x slower.  Reading the first
    // chunk's y speculatively before the wait measured no faster and costs 8 registers —
    // above 32 the persistent grid loses occupancy: 1.24 -> 1.35 ms.)
    if (d.grid_wait) {
      const int cr = crit[idx];
      if (lane == 0 && cr >= 0) wait_value(&ysrc[cr], d.poll_ns);
      __syncwarp();
    }
    for (int c0 = beg; c0 < end; c0 += 32) {
      const int cnt = min(32, end - c0);
      double p = 0.0;
      int ncol = 0;
      double nv = 0.0;
      if (c0 + 32 + lane < end) {
        ncol = ci[c0 + 32 + lane];
        nv = vals[c0 + 32 + lane];
      }
      if (lane < cnt) p = __dmul_rn(v, wait_value(&ysrc[col], d.poll_ns));
      for (int i = 0; i < cnt; ++i) acc = __dsub_rn(acc, __shfl_sync(0xffffffffu, p, i));
      col = ncol;
      v = nv;
    }
    if (lane == 0) {
      double w = acc;
      if (IS_U) w = __ddiv_rn(acc, piv);
      st_relaxed_f64(&ysrc[r], unsentinel(w));  // publish first: other rows wait on it
      if (d.trace_trsv && sys == 0) d.trace_trsv[(IS_U ? d.n : 0) + r] = globaltimer();
      st_relaxed_f64(&yres[r], __longlong_as_double((long long)SENTINEL_BITS));
      if (IS_U) {
        xout[(size_t)sys * d.n + d.col_perm[r]] = w;
        if (!isfinite(w)) atomicOr(&d.scal[(size_t)sys * SCAL_STRIDE + SC_NONFINITE], 1ull);
      }
    }
  }
}

// ---- grid phase as chain tasks (single system; plan.cpp build_chains) ---------------------
// Task codes: r (one row, as k_trsv_grid), -(r+1) (the external prefix of chain row r, into
// cpart), r0 | (m-1) << 26 (a chain of m rows r0, r0 +- 1, ...).  The per-row arithmetic is
// k_trsv_grid's: the prefix is summed in CSR order from the row's initial value, and the chain
// warp continues each row with its internal entries in CSR order (lane i = row i; the column
// of step j is row j of the chain, so consuming entries as the steps come keeps that order).
// One-row and prefix tasks: lane 0 waits on the critical dependency, the lanes then sum the
// entries [beg, end) 32 at a time, in order, from `acc` (uniform across the warp).
template <bool IS_U>
__device__ __forceinline__ double chain_row_sum(const DevPlan &d, const int *__restrict__ ci,
                                                const double *__restrict__ vals, const double *ysrc,
                                                int beg, int end, int cr, double acc, int lane) {
  int col = 0;
  double v = 0.0;
  if (beg + lane < end) {
    col = ci[beg + lane];
    v = vals[beg + lane];
  }
  if (lane == 0 && cr >= 0) wait_value(&ysrc[cr], d.poll_ns);
  __syncwarp();
  for (int c0 = beg; c0 < end; c0 += 32) {
    const int cnt = min(32, end - c0);
    double p = 0.0;
    int ncol = 0;
    double nv = 0.0;
    if (c0 + 32 + lane < end) {
      ncol = ci[c0 + 32 + lane];
      nv = vals[c0 + 32 + lane];
    }
    if (lane < cnt) p = __dmul_rn(v, wait_value(&ysrc[col], d.poll_ns));
    for (int i = 0; i < cnt; ++i) acc = __dsub_rn(acc, __shfl_sync(0xffffffffu, p, i));
    col = ncol;
    v = nv;
  }
  return acc;
}

template <bool IS_U>
__global__ void __launch_bounds__(256, 8) k_trsv_chain(DevPlan d, const double *__restrict__ b,
                                                    double *__restrict__ xout) {
  if (!sys_active(d, 0)) return;
  const int lane = threadIdx.x & 31;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int *task = IS_U ? d.Uc_task : d.Lc_task;
  const int *aux = IS_U ? d.Uc_aux : d.Lc_aux;
  const int *split = IS_U ? d.Uc_split : d.Lc_split;
  const int ntask = IS_U ? d.nUc : d.nLc;
  const int *rp = IS_U ? d.Urp : d.Lrp;
  const int *ci = IS_U ? d.Uci : d.Lci;
  const double *vals = IS_U ? d.Uv : d.Lv;
  double *ysrc = IS_U ? d.yU : d.yL;  // published by this sweep
  double *yres = IS_U ? d.yL : d.yU;  // reset for the next solve
  for (int idx = gwarp; idx < ntask; idx += nwarps) {
    const int code = task[idx], ax = aux[idx];
    if (code < 0 || (code >> 26) == 0) {  // one row, or a chain row's external prefix
      const bool prefix = code < 0;
      const int r = prefix ? -code - 1 : code;
      const int beg = IS_U ? d.Ugrid_split[r] : rp[r];
      const int end = prefix ? split[r] : rp[r + 1];
      const double init = IS_U ? ldcg(&d.yL[r]) : b[d.row_perm[r]];
      const double piv = (IS_U && !prefix) ? d.udiag[r] : 1.0;
      const double acc = chain_row_sum<IS_U>(d, ci, vals, ysrc, beg, end, ax, init, lane);
      if (lane == 0) {
        if (prefix) st_relaxed_f64(&d.cpart[r], unsentinel(acc));
        else {
          const double w = IS_U ? __ddiv_rn(acc, piv) : acc;
          st_relaxed_f64(&ysrc[r], unsentinel(w));
          if (d.trace_trsv) d.trace_trsv[(IS_U ? d.n : 0) + r] = globaltimer();
          st_relaxed_f64(&yres[r], __longlong_as_double((long long)SENTINEL_BITS));
          if (IS_U) {
            xout[d.col_perm[r]] = w;
            if (!isfinite(w)) atomicOr(&d.scal[SC_NONFINITE], 1ull);
          }
        }
      }
      continue;
    }
    const int r0 = code & ((1 << 26) - 1), m = (code >> 26) + 1;
    const int r = IS_U ? r0 - lane : r0 + lane;
    const bool act = lane < m;
    double piv = 1.0, acc = 0.0, cv = 0.0;
    int q = 0, qe = 0, cc = -1;
    if (act) {
      q = split[r];
      qe = rp[r + 1];
      if (IS_U) piv = d.udiag[r];
      if (q < qe) {
        cc = ci[q];
        cv = vals[q];
      }
      if ((ax >> lane) & 1) {  // the prefix task's sum (then reset for the next solve)
        acc = wait_value(&d.cpart[r], d.poll_ns);
        d.cpart[r] = __longlong_as_double((long long)SENTINEL_BITS);
      } else {
        acc = IS_U ? ldcg(&d.yL[r]) : b[d.row_perm[r]];
      }
    }
    // Per step only the publish of y_j is on the chain; the other buffer's reset and x (U) are
    // written after the loop.  (Measured: staging the internal entries in shared memory, or a
    // branch-free step with a consumption bit mask, is no faster — the step is bound by the
    // warps sharing the SM: ~1,000 cycles per row at 64 warps per SM, ~400 at 16.)
    const long long t_loop = d.trace_step ? clock64() : 0;
    double mine = 0.0;
    for (int j = 0; j < m; ++j) {
      const double w = IS_U ? __ddiv_rn(acc, piv) : acc;
      const double yj = __shfl_sync(0xffffffffu, w, j);
      if (lane == j) {
        st_relaxed_f64(&ysrc[r], unsentinel(yj));  // publish first: other rows wait on it
        mine = yj;
      }
      if (cc == (IS_U ? r0 - j : r0 + j)) {  // this row's next internal entry is column r_j
        acc = __dsub_rn(acc, __dmul_rn(cv, yj));
        cc = -1;
        if (++q < qe) {
          cc = ci[q];
          cv = vals[q];
        }
      }
    }
    if (act) {
      if (d.trace_trsv) d.trace_trsv[(IS_U ? d.n : 0) + r] = globaltimer();
      st_relaxed_f64(&yres[r], __longlong_as_double((long long)SENTINEL_BITS));
      if (IS_U) {
        xout[d.col_perm[r]] = mine;
        if (!isfinite(mine)) atomicOr(&d.scal[SC_NONFINITE], 1ull);
      }
    }
    const size_t to = 2 * (size_t)idx + (IS_U ? 2 * (size_t)d.n : 0);
    if (d.trace_step && !d.trace_trsv && lane == 0 && to + 1 < 4 * (size_t)d.n) {
      d.trace_step[to] = (unsigned long long)m;  // KKT_TRACE=2: {rows, loop cycles}
      d.trace_step[to + 1] = (unsigned long long)(clock64() - t_loop);
    }
  }
}

cudaError_t launch_trsv_chain(const DevPlan &d, bool upper, const double *b, double *x, int grid_blocks,
                              cudaStream_t s) {
  if (upper) k_trsv_chain<true><<<grid_blocks, 256, 0, s>>>(d, b, x);
  else k_trsv_chain<false><<<grid_blocks, 256, 0, s>>>(d, b, x);
  return cudaGetLastError();
}

// ---- row-parallel launches: rows whose dependencies are all final (an earlier launch) ------
// Thread per (row, system) — for a batch 32+ consecutive threads are the systems of one row,
// so every value access is coalesced.  Used for the wide leading L levels (no waiting at
// all) and for the tail rows' leading partial sums (PARTIAL: into tacc, seeding the sweep).
template <bool IS_U, bool PARTIAL>
__global__ void __launch_bounds__(256) k_trsv_rows(DevPlan d, const int *__restrict__ rows, int count,
                                                   const double *__restrict__ b,
                                                   double *__restrict__ xout) {
  const int *rp = IS_U ? d.Urp : d.Lrp;
  const int *ci = IS_U ? d.Uci : d.Lci;
  const double *vals = IS_U ? d.Uv : d.Lv;
  double *ysrc = IS_U ? d.yU : d.yL;
  double *yres = IS_U ? d.yL : d.yU;
  const int64_t total = (int64_t)count * d.nbp;
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < total;
       f += (int64_t)gridDim.x * blockDim.x) {
    const int idx = (int)(f / d.nbp), sys = (int)(f - (int64_t)idx * d.nbp);
    if (!sys_active(d, sys)) continue;
    const int r = rows[idx];
    const int beg = rp[r];
    const int end = PARTIAL ? (IS_U ? d.Ugrid_split[r] : d.Ltail_split[r - d.pL]) : rp[r + 1];
    double acc = IS_U ? ldcg(&d.yL[IL(d, r, sys)]) : b[IL(d, d.row_perm[r], sys)];
    for (int c0 = beg; c0 < end; c0 += 4) {
      double v[4], y[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (c0 + q < end) {
          v[q] = vals[IL(d, c0 + q, sys)];
          y[q] = ldcg(&ysrc[IL(d, ci[c0 + q], sys)]);
        }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (c0 + q < end) acc = __dsub_rn(acc, __dmul_rn(v[q], y[q]));
    }
    if (PARTIAL) {
      if (IS_U) d.yL[IL(d, r, sys)] = acc;  // the grid row resumes from here (Ugrid_split)
      else d.tacc[IL(d, r - d.pL, sys)] = acc;
      continue;
    }
    const double w = IS_U ? __ddiv_rn(acc, d.udiag[IL(d, r, sys)]) : acc;
    ysrc[IL(d, r, sys)] = unsentinel(w);
    yres[IL(d, r, sys)] = __longlong_as_double((long long)SENTINEL_BITS);
    if (IS_U) {
      xout[IL(d, d.col_perm[r], sys)] = w;
      if (!isfinite(w)) atomicOr(&d.scal[(size_t)sys * SCAL_STRIDE + SC_NONFINITE], 1ull);
    }
  }
}

cudaError_t launch_trsv_rows(const DevPlan &d, bool partial, const int *rows, int count,
                             const double *b, double *x, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  const int64_t total = (int64_t)count * d.nbp;
  const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, 16 * 148);
  if (partial) k_trsv_rows<false, true><<<grid, 256, 0, s>>>(d, rows, count, b, x);
  else k_trsv_rows<false, false><<<grid, 256, 0, s>>>(d, rows, count, b, x);
  return cudaGetLastError();
}

cudaError_t launch_U_partial(const DevPlan &d, cudaStream_t s, long long *launches) {
  if (!d.u_partial || d.n_upart <= 0) return cudaSuccess;
  const int64_t total = (int64_t)d.n_upart * d.nbp;
  const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, 16 * 148);
  k_trsv_rows<true, true><<<grid, 256, 0, s>>>(d, d.U_part_rows, d.n_upart, nullptr, nullptr);
  ++*launches;
  return cudaGetLastError();
}

// the L phase before the sweep: row-parallel leading levels, the sync-free grid kernel for
// the rest (launch_grid), then the tail rows' partial sums
cudaError_t launch_L_front(const DevPlan &d, const double *b, double *x, int grid_blocks, cudaStream_t s,
                           long long *launches) {
  cudaError_t e = cudaSuccess;
  for (int l = 0; l < d.L_nsync && e == cudaSuccess; ++l) {
    e = launch_trsv_rows(d, false, d.L_grid_order + d.L_sync_ptr[l], d.L_sync_ptr[l + 1] - d.L_sync_ptr[l],
                         b, x, s);
    ++*launches;
  }
  if (e == cudaSuccess && d.nLg > d.L_sync_ptr[d.L_nsync]) {
    if (d.nbp > 1) {
      e = b_launch_grid_L(d, b, x, grid_blocks, s);
    } else if (d.chains) {
      e = launch_trsv_chain(d, false, b, x, grid_blocks, s);
    } else {
      k_trsv_grid<false><<<grid_blocks, 256, 0, s>>>(d, b, x);
      e = cudaGetLastError();
    }
    ++*launches;
  }
  if (e == cudaSuccess && d.n > d.pL) {
    e = launch_trsv_rows(d, true, d.L_tail_order, d.n - d.pL, b, x, s);
    ++*launches;
  }
  return e;
}

// x += y (numpy's elementwise add, one rounding)
__global__ void k_add_inplace(double *__restrict__ x, const double *__restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = __dadd_rn(x[i], y[i]);
}

cudaError_t launch_add_inplace(double *x, const double *y, int64_t n, cudaStream_t s) {
  if (n > 0) k_add_inplace<<<(unsigned)std::min<int64_t>((n + 255) / 256, 8 * 148), 256, 0, s>>>(x, y, n);
  return cudaGetLastError();
}

__global__ void k_fill_sentinel(double *p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = __longlong_as_double((long long)SENTINEL_BITS);
}

cudaError_t launch_fill_sentinel(double *p, int64_t n, cudaStream_t s) {
  if (n) k_fill_sentinel<<<148, 256, 0, s>>>(p, n);
  return cudaGetLastError();
}

cudaError_t trsv_configure(int *grid_blocks_per_sm) {
  int a = 0, b = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_trsv_grid<false>, 256, 0);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_trsv_grid<true>, 256, 0);
  int c = 0, u = 0;  // the chain kernels run on the same persistent grid
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, k_trsv_chain<false>, 256, 0);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&u, k_trsv_chain<true>, 256, 0);
  if (e != cudaSuccess) return e;
  *grid_blocks_per_sm = std::min(std::min(a, b), std::min(c, u));
  return e;
}

cudaError_t launch_trsv(const DevPlan &d, const double *b, double *x, int grid_blocks,
                        cudaStream_t s, long long *launches) {
  if (!d.n) return cudaSuccess;
  const int TL = d.n - d.pL, TU = d.n - d.pU;
  {  // forward: grid rows, then the sweep over the trailing block
    cudaError_t e = launch_L_front(d, b, x, grid_blocks, s, launches);
    if (e != cudaSuccess) return e;
  }
  if (TL) {
    cudaError_t e = launch_sweep_blocked(d, false, x, s);
    if (e != cudaSuccess) return e;
    ++*launches;
  }
  if (TU) {  // backward: the sweep over the trailing block, then the grid rows
    cudaError_t e = launch_sweep_blocked(d, true, x, s);
    if (e != cudaSuccess) return e;
    ++*launches;
  }
  if (d.nUg) {
    cudaError_t e = launch_U_partial(d, s, launches);
    if (e != cudaSuccess) return e;
    if (d.chains) launch_trsv_chain(d, true, b, x, grid_blocks, s);
    else k_trsv_grid<true><<<grid_blocks, 256, 0, s>>>(d, b, x);
    ++*launches;
  }
  return cudaGetLastError();
}

}  // namespace kkt
