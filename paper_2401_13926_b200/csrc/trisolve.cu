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
//     replays the reference's own column sweep over the block in shared memory: per column
//     one barrier, each target updated by one thread.  Column data stream in through a
//     cp.async ring RING-1 columns ahead, so a step costs a barrier + a shared RMW.
//   L = [grid rows < pL] then [sweep columns pL..n-1];
//   U = [sweep columns n-1..pU] then [grid rows < pU].
// Each sweep resets the other sweep's buffer for the next solve, so no memsets are needed.
#include <cuda_runtime.h>

#include "device.h"
#include "kernels.cuh"

namespace kkt {

constexpr int SWEEP_THREADS = 128;  // 4 warps: cheap barrier, <= 2 entries per thread per step



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
  // task = (level-ordered row index, system): row-major so all systems' copies of a row
  // are adjacent and every dependency of a task has a smaller task index
  for (int task = gwarp; task < ntask; task += nwarps) {
    const int idx = task / d.nb, sys = task % d.nb;
    if (!sys_active(d, sys)) continue;
    const int r = order[idx];
    const double *vals = (IS_U ? d.Uv : d.Lv) + (size_t)sys * nnz;
    double *ysrc = (IS_U ? d.yU : d.yL) + (size_t)sys * d.n;  // published by this sweep
    double *yres = (IS_U ? d.yL : d.yU) + (size_t)sys * d.n;  // reset for the next solve
    // L: rows >= pL are the sweep block's rows; here only their leading entries (columns
    // < pL) are summed, into tacc, which seeds the sweep (same per-row order).
    const bool partial = !IS_U && r >= d.pL;
    const int beg = rp[r], end = partial ? d.Ltail_split[r - d.pL] : rp[r + 1];
    // independent loads first: the initial value and the first chunk's pattern/values
    double acc = IS_U ? ldcg(&d.yL[(size_t)sys * d.n + r]) : b[(size_t)sys * d.n + d.row_perm[r]];
    const double piv = IS_U ? d.udiag[(size_t)sys * d.n + r] : 1.0;  // off the critical path
    int col = 0;
    double v = 0.0;
    if (beg + lane < end) {
      col = ci[beg + lane];
      v = vals[beg + lane];
    }
    // lane 0 alone spins on the critical dependency; the other dependencies are then
    // normally published already, so the lanes' loads below rarely have to wait
    const int cr = crit[idx];
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
    if (lane == 0) {
      double w = acc;
      if (partial) {
        d.tacc[(size_t)sys * (d.n - d.pL) + r - d.pL] = acc;
        continue;
      }
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

// ---- sweep phase: one CTA, the reference's column sweep on the dense separator block --------
template <bool IS_U, int RING, int SLOT>
__global__ void __launch_bounds__(SWEEP_THREADS) k_trsv_sweep(DevPlan d,
                                                              const double *__restrict__ b,
                                                              double *__restrict__ xout) {
  extern __shared__ double sm[];
  const int sys = blockIdx.x;  // one CTA per system: the nb sweeps run side by side
  if (!sys_active(d, sys)) return;
  const int p = IS_U ? d.pU : d.pL;
  const int T = d.n - p;
  const int tid = threadIdx.x;
  double *acc = sm;                                           // [T]
  double *dg = acc + T;                                       // [T] (U: pivots)
  double *rv = dg + (IS_U ? T : 0);                           // [RING*SLOT] values
  int *rr = reinterpret_cast<int *>(rv + RING * SLOT);  // [RING*SLOT] rows
  int *cbeg = rr + RING * SLOT;                   // [T] CSC range of step s
  int *cend = cbeg + T;                                       // [T]
  int *cperm = cend + T;                                      // [T] (U: col_perm)
  const double *cvals = (IS_U ? d.Ux : d.Lx) + (size_t)sys * (IS_U ? d.nnz_U : d.nnz_L);
  const int *crows = IS_U ? d.Ui : d.Li;
  double *yL = d.yL + (size_t)sys * d.n;
  double *yU = d.yU + (size_t)sys * d.n;
  xout += (size_t)sys * d.n;
  // step s handles column j(s): L ascending from p, U descending from n-1
  for (int s = tid; s < T; s += blockDim.x) {
    const int j = IS_U ? d.n - 1 - s : p + s;
    cbeg[s] = IS_U ? d.Up[j] + d.Uhead_off[j - p] : d.Lp[j];
    cend[s] = IS_U ? d.Up[j + 1] : d.Lp[j + 1];
    if (IS_U) {
      dg[j - p] = d.udiag[(size_t)sys * d.n + j];
      cperm[s] = d.col_perm[j];
    }
  }
  if (IS_U) {
    // acc = L result of the head rows; reset yL for the next solve
    for (int r = p + tid; r < d.n; r += blockDim.x) {
      acc[r - p] = ldcg(&yL[r]);
      yL[r] = __longlong_as_double((long long)SENTINEL_BITS);
    }
  } else {
    // acc_r = b_perm[r] - sum_{j < p} L(r,j) y_j (ascending j) was computed by the grid
    // kernel as the partial rows; reset yU for the next solve.
    const double *ta = d.tacc + (size_t)sys * T;
    for (int r = p + tid; r < d.n; r += blockDim.x) {
      acc[r - p] = ldcg(&ta[r - p]);
      yU[r] = __longlong_as_double((long long)SENTINEL_BITS);
    }
  }
  __syncthreads();
  auto issue = [&](int s) {
    if (s < T) {
      const int slot = s % RING;
      const int beg = cbeg[s], cnt = min(cend[s] - beg, SLOT);
      for (int e = tid; e < cnt; e += blockDim.x) {
        cp_async8(&rv[slot * SLOT + e], &cvals[beg + e]);
        cp_async4(&rr[slot * SLOT + e], &crows[beg + e]);
      }
    }
    cp_async_commit();
  };
#pragma unroll 1
  for (int s = 0; s < RING - 1; ++s) issue(s);
  bool bad = false;
#pragma unroll 1
  for (int s = 0; s < T; ++s) {
    cp_async_wait<RING - 2>();
    __syncthreads();
    issue(s + RING - 1);
    const int j = IS_U ? d.n - 1 - s : p + s;
    double yj = acc[j - p];
    if (IS_U) yj = __ddiv_rn(yj, dg[j - p]);
    if (tid == 0) {
      const double w = unsentinel(yj);
      if (IS_U) {
        yU[j] = w;
        xout[cperm[s]] = yj;
        if (!isfinite(yj)) bad = true;
      } else {
        yL[j] = w;
      }
    }
    const int slot = s % RING;
    const int beg = cbeg[s], cnt = cend[s] - beg;
    for (int e = tid; e < cnt; e += blockDim.x) {
      double v;
      int r;
      if (e < SLOT) {
        v = rv[slot * SLOT + e];
        r = rr[slot * SLOT + e];
      } else {
        v = cvals[beg + e];
        r = crows[beg + e];
      }
      acc[r - p] = __dsub_rn(acc[r - p], __dmul_rn(v, yj));
    }
  }
  cp_async_wait<0>();
  if (IS_U && bad) atomicOr(&d.scal[(size_t)sys * SCAL_STRIDE + SC_NONFINITE], 1ull);
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

// ring shapes (RING x SLOT entries, 96 KB each): deep rings for short columns
constexpr int RING_BYTES = 96 * 1024;
static size_t sweep_smem(int T, bool upper) {
  return (size_t)T * 8 * (upper ? 2 : 1) + (size_t)RING_BYTES + (size_t)T * 12;
}

template <bool IS_U>
static cudaError_t configure_sweep() {
  const int sm = (int)sweep_smem(KKT_CTA_PHASE_MAX_ROWS, IS_U);
  cudaError_t e = cudaFuncSetAttribute(k_trsv_sweep<IS_U, 32, 256>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_trsv_sweep<IS_U, 16, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_trsv_sweep<IS_U, 8, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  return e;
}

template <bool IS_U>
static void launch_sweep(const DevPlan &d, const double *b, double *x, int T, int maxcol,
                         cudaStream_t s) {
  const size_t sm = sweep_smem(T, IS_U);
  if (maxcol <= 256)
    k_trsv_sweep<IS_U, 32, 256><<<d.nb, SWEEP_THREADS, sm, s>>>(d, b, x);
  else if (maxcol <= 512)
    k_trsv_sweep<IS_U, 16, 512><<<d.nb, SWEEP_THREADS, sm, s>>>(d, b, x);
  else
    k_trsv_sweep<IS_U, 8, 1024><<<d.nb, SWEEP_THREADS, sm, s>>>(d, b, x);
}

cudaError_t trsv_configure(int *grid_blocks_per_sm) {
  int a = 0, b = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_trsv_grid<false>, 256, 0);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_trsv_grid<true>, 256, 0);
  if (e != cudaSuccess) return e;
  *grid_blocks_per_sm = a < b ? a : b;
  e = configure_sweep<false>();
  if (e == cudaSuccess) e = configure_sweep<true>();
  return e;
}

cudaError_t launch_trsv(const DevPlan &d, const double *b, double *x, int grid_blocks,
                        cudaStream_t s, long long *launches) {
  if (!d.n) return cudaSuccess;
  const int TL = d.n - d.pL, TU = d.n - d.pU;
  if (d.nLg) {  // forward: grid rows, then the sweep over the trailing block
    k_trsv_grid<false><<<grid_blocks, 256, 0, s>>>(d, b, x);
    ++*launches;
  }
  if (TL) {
    launch_sweep<false>(d, b, x, TL, d.sweep_maxL, s);
    ++*launches;
  }
  if (TU) {  // backward: the sweep over the trailing block, then the grid rows
    launch_sweep<true>(d, b, x, TU, d.sweep_maxU, s);
    ++*launches;
  }
  if (d.nUg) {
    k_trsv_grid<true><<<grid_blocks, 256, 0, s>>>(d, b, x);
    ++*launches;
  }
  return cudaGetLastError();
}

}  // namespace kkt
