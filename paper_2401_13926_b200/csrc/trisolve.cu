// Triangular solves x = lu_solve(b) (direct_lu.py:359-379), bitwise with the reference.
//
// The reference sweeps columns: forward `y[Li(j)] -= Lx(j)*y[j]` for ascending j, backward
// `y_j /= u_jj; y[Ui(j)] -= Ux(j)*y_j` for descending j.  Row r therefore receives its
// updates in ascending column order (L) / descending column order (U); a row-oriented solve
// that accumulates each CSR row sequentially in that order, with separately rounded products,
// reproduces every bit.
//
// Schedule (per sweep, chosen on the host from the level profile, plan.cpp choose_tail):
//   * grid phase — persistent, sync-free, warp per row, rows round-robin in level order.
//     Readiness is the value itself: y is reset to a sentinel NaN pattern and a consumer
//     re-reads y[col] until it is published (one L2 round trip per dependency hop);
//   * CTA phase — the narrow end of the DAG (the dense separator rows at the end of the
//     elimination order): one 1024-thread CTA, thread per row, y of the phase rows in shared
//     memory with the same sentinel protocol (~40 cycles per hop instead of ~1 us).
//   L = [grid rows < pL] then [CTA rows >= pL];  U = [CTA rows >= pU] then [grid rows < pU].
// Each sweep resets the other sweep's buffer for the next solve, so no memsets are needed.
#include <cuda_runtime.h>

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
  const int nrows = IS_U ? d.nUg : d.nLg;
  const int *rp = IS_U ? d.Urp : d.Lrp;
  const int *ci = IS_U ? d.Uci : d.Lci;
  const double *vals = IS_U ? d.Uv : d.Lv;
  double *ysrc = IS_U ? d.yU : d.yL;  // dependencies (published by this sweep)
  double *yres = IS_U ? d.yL : d.yU;  // the other sweep's buffer: reset for the next solve
  bool bad = false;
  for (int idx = gwarp; idx < nrows; idx += nwarps) {
    const int r = order[idx];
    double acc;
    if (IS_U) {
      acc = ldcg(&d.yL[r]);  // final L result (previous kernel)
    } else {
      acc = b[d.row_perm[r]];
    }
    const int beg = rp[r], end = rp[r + 1];
    // prefetch the first chunk's pattern/values (independent of the dependencies)
    int col = 0;
    double v = 0.0;
    if (beg + lane < end) {
      col = ci[beg + lane];
      v = vals[beg + lane];
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
      if (lane < cnt) p = __dmul_rn(v, wait_value(&ysrc[col]));
      for (int i = 0; i < cnt; ++i) acc = __dsub_rn(acc, __shfl_sync(0xffffffffu, p, i));
      col = ncol;
      v = nv;
    }
    if (lane == 0) {
      double w = acc;
      if (IS_U) {
        w = __ddiv_rn(acc, d.udiag[r]);
        xout[d.col_perm[r]] = w;
        if (!isfinite(w)) bad = true;
      }
      st_relaxed_f64(&yres[r], __longlong_as_double((long long)SENTINEL_BITS));
      st_relaxed_f64(&ysrc[r], unsentinel(w));
    }
  }
  if (IS_U && bad) atomicOr(&d.scal[SC_NONFINITE], 1ull);
}

// ---- CTA phase: one block, thread per row, phase rows' y in shared memory ----------------
template <bool IS_U>
__global__ void __launch_bounds__(CTA_PHASE_THREADS) k_trsv_cta(DevPlan d,
                                                                const double *__restrict__ b,
                                                                double *__restrict__ xout) {
  extern __shared__ double ys[];  // rows [p, n) -> slot r - p
  const int p = IS_U ? d.pU : d.pL;
  const int T = d.n - p;
  const int *order = IS_U ? d.U_head_order : d.L_tail_order;
  const int *rp = IS_U ? d.Urp : d.Lrp;
  const int *ci = IS_U ? d.Uci : d.Lci;
  const double *vals = IS_U ? d.Uv : d.Lv;
  double *ysrc = IS_U ? d.yU : d.yL;
  double *yres = IS_U ? d.yL : d.yU;
  volatile double *vys = ys;
  for (int s = threadIdx.x; s < T; s += blockDim.x) ys[s] = __longlong_as_double((long long)SENTINEL_BITS);
  __syncthreads();
  bool bad = false;
  for (int idx = threadIdx.x; idx < T; idx += blockDim.x) {
    const int r = order[idx];
    double acc = IS_U ? ldcg(&d.yL[r]) : b[d.row_perm[r]];
    const int beg = rp[r], end = rp[r + 1];
    for (int e = beg; e < end; ++e) {
      const int col = ci[e];
      const double v = vals[e];
      double y;
      if (col >= p) {
        y = vys[col - p];
        while (is_sentinel(y)) y = vys[col - p];
      } else {
        y = ldcg(&ysrc[col]);  // grid phase of this sweep already complete (L only)
      }
      acc = __dsub_rn(acc, __dmul_rn(v, y));
    }
    double w = acc;
    if (IS_U) {
      w = __ddiv_rn(acc, d.udiag[r]);
      xout[d.col_perm[r]] = w;
      if (!isfinite(w)) bad = true;
    }
    w = unsentinel(w);
    yres[r] = __longlong_as_double((long long)SENTINEL_BITS);
    ysrc[r] = w;
    vys[r - p] = w;
  }
  if (IS_U && bad) atomicOr(&d.scal[SC_NONFINITE], 1ull);
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
  if (e != cudaSuccess) return e;
  *grid_blocks_per_sm = a < b ? a : b;
  const int smem = KKT_CTA_PHASE_MAX_ROWS * 8;
  e = cudaFuncSetAttribute(k_trsv_cta<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_trsv_cta<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  return e;
}

cudaError_t launch_trsv(const DevPlan &d, const double *b, double *x, int grid_blocks,
                        cudaStream_t s, long long *launches) {
  if (!d.n) return cudaSuccess;
  const size_t smL = 8 * (size_t)(d.n - d.pL), smU = 8 * (size_t)(d.n - d.pU);
  // forward: grid rows then the CTA tail
  if (d.nLg) {
    k_trsv_grid<false><<<grid_blocks, 256, 0, s>>>(d, b, x);
    ++*launches;
  }
  if (d.n > d.pL) {
    k_trsv_cta<false><<<1, CTA_PHASE_THREADS, smL, s>>>(d, b, x);
    ++*launches;
  }
  // backward: CTA head then the grid rows
  if (d.n > d.pU) {
    k_trsv_cta<true><<<1, CTA_PHASE_THREADS, smU, s>>>(d, b, x);
    ++*launches;
  }
  if (d.nUg) {
    k_trsv_grid<true><<<grid_blocks, 256, 0, s>>>(d, b, x);
    ++*launches;
  }
  return cudaGetLastError();
}

}  // namespace kkt
