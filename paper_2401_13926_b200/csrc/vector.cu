// Memory-bound vector kernels of the operator: SpMV (sparsecore.spmv, sparsecore.py:284-305)
// in the reference's accumulation order, and the fused residual statistics behind
// refine.nsr / nrbe / needs_refinement (refine.py:62-92).  Reductions use a fixed grid and a
// fixed-shape tree, so results are run-to-run deterministic.
#include <cuda_runtime.h>

#include "device.h"
#include "kernels.cuh"

namespace kkt {

// ============================================================================
// SpMV y = K x in the reference accumulation order.  Symmetric-lower input: the
// reference sums the stored lower row (cols <= i, ascending) and, separately, the mirrored
// strict entries (rows k > i ascending) and adds the two bincounts; in the expanded
// general row these are the two halves split at the diagonal.  Optional r = b - y.
// Also accumulates ||out||^2 partials when `nrm` is given (deterministic 2-stage).
// ============================================================================
__global__ void __launch_bounds__(RED_THREADS) k_spmv(DevPlan d, const double *__restrict__ x,
                                                      double *__restrict__ out,
                                                      const double *__restrict__ bsub,
                                                      double *__restrict__ nrm_out) {
  __shared__ double sh[32];
  double loc = 0.0;
  bool bad = false;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d.n; i += gridDim.x * blockDim.x) {
    const int b = d.A_rp[i], s = d.A_split[i], e = d.A_rp[i + 1];
    double s1 = 0.0, s2 = 0.0, y;
    if (d.sym_lower) {
      for (int p = b; p < s; ++p) s1 = __dadd_rn(s1, __dmul_rn(d.A_vals[p], x[d.A_ci[p]]));
      for (int p = s; p < e; ++p) s2 = __dadd_rn(s2, __dmul_rn(d.A_vals[p], x[d.A_ci[p]]));
      y = __dadd_rn(s1, s2);
    } else {
      for (int p = b; p < e; ++p) s1 = __dadd_rn(s1, __dmul_rn(d.A_vals[p], x[d.A_ci[p]]));
      y = s1;
    }
    if (!isfinite(y)) bad = true;
    const double o = bsub ? __dsub_rn(bsub[i], y) : y;
    out[i] = o;
    loc = __dadd_rn(loc, __dmul_rn(o, o));
  }
  if (bad) atomicOr(&d.scal[SC_NONFINITE], 1ull);
  if (nrm_out) {
    const double t = block_sum<RED_THREADS>(loc, sh);
    if (threadIdx.x == 0) nrm_out[blockIdx.x] = t;
  }
}

// Final ordered reduction of RED_BLOCKS partials (one warp, fixed order).
__global__ void k_reduce_partials(const double *__restrict__ partials, int nvec, int nblk,
                                  double *__restrict__ out, int op_sqrt) {
  const int v = blockIdx.x;
  if (v >= nvec) return;
  double s = 0.0;
  for (int b = threadIdx.x; b < nblk; b += 32) s += partials[(size_t)v * nblk + b];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) out[v] = op_sqrt ? sqrt(s) : s;
}

// ============================================================================
// Residual statistics for (r, x):  e = r - K x  (spmv order), then
// {||e||_2^2, max|e|, ||x||_2^2, max|x|, ||r||_2^2} partials.
// ============================================================================
__global__ void __launch_bounds__(RED_THREADS) k_resid_stats(DevPlan d, const double *__restrict__ r,
                                                             const double *__restrict__ x,
                                                             double *__restrict__ partials) {
  __shared__ double sh[32];
  double e2 = 0.0, emax = 0.0, x2 = 0.0, xmax = 0.0, r2 = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d.n; i += gridDim.x * blockDim.x) {
    const int b = d.A_rp[i], s = d.A_split[i], e = d.A_rp[i + 1];
    double s1 = 0.0, s2 = 0.0, y;
    if (d.sym_lower) {
      for (int p = b; p < s; ++p) s1 = __dadd_rn(s1, __dmul_rn(d.A_vals[p], x[d.A_ci[p]]));
      for (int p = s; p < e; ++p) s2 = __dadd_rn(s2, __dmul_rn(d.A_vals[p], x[d.A_ci[p]]));
      y = __dadd_rn(s1, s2);
    } else {
      for (int p = b; p < e; ++p) s1 = __dadd_rn(s1, __dmul_rn(d.A_vals[p], x[d.A_ci[p]]));
      y = s1;
    }
    const double ei = __dsub_rn(r[i], y);
    e2 += ei * ei;
    emax = fmax(emax, fabs(ei));
    x2 += x[i] * x[i];
    xmax = fmax(xmax, fabs(x[i]));
    r2 += r[i] * r[i];
  }
  double t;
  t = block_sum<RED_THREADS>(e2, sh);
  if (threadIdx.x == 0) partials[0 * RED_BLOCKS + blockIdx.x] = t;
  t = block_sum<RED_THREADS>(x2, sh);
  if (threadIdx.x == 0) partials[2 * RED_BLOCKS + blockIdx.x] = t;
  t = block_sum<RED_THREADS>(r2, sh);
  if (threadIdx.x == 0) partials[4 * RED_BLOCKS + blockIdx.x] = t;
  // maxima: warp/block max then partial
  emax = warp_max(emax);
  xmax = warp_max(xmax);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    sh[threadIdx.x >> 5] = emax;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < RED_THREADS / 32; ++w) m = fmax(m, sh[w]);
    partials[1 * RED_BLOCKS + blockIdx.x] = m;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = xmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < RED_THREADS / 32; ++w) m = fmax(m, sh[w]);
    partials[3 * RED_BLOCKS + blockIdx.x] = m;
  }
}

__global__ void k_resid_final(const double *__restrict__ partials, double *__restrict__ out) {
  // out: {||e||_2, ||e||_inf, ||x||_2, ||x||_inf, ||r||_2}
  const int v = blockIdx.x;
  double s = 0.0;
  const bool is_max = (v == 1 || v == 3);
  for (int b = threadIdx.x; b < RED_BLOCKS; b += 32) {
    const double p = partials[v * RED_BLOCKS + b];
    s = is_max ? fmax(s, p) : s + p;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double q = __shfl_down_sync(0xffffffffu, s, o);
    s = is_max ? fmax(s, q) : s + q;
  }
  if (threadIdx.x == 0) out[v] = is_max ? s : sqrt(s);
}


cudaError_t launch_spmv(const DevPlan &d, const double *x, double *out, const double *bsub,
                        double *nrm_partials, cudaStream_t s) {
  k_spmv<<<RED_BLOCKS, RED_THREADS, 0, s>>>(d, x, out, bsub, nrm_partials);
  return cudaGetLastError();
}

cudaError_t launch_reduce_partials(const double *partials, int nvec, int nblk, double *out,
                                   int op_sqrt, cudaStream_t s) {
  k_reduce_partials<<<nvec, 32, 0, s>>>(partials, nvec, nblk, out, op_sqrt);
  return cudaGetLastError();
}

cudaError_t launch_resid_stats(const DevPlan &d, const double *r, const double *x,
                               double *partials, double *out5, cudaStream_t s) {
  k_resid_stats<<<RED_BLOCKS, RED_THREADS, 0, s>>>(d, r, x, partials);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_resid_final<<<5, 32, 0, s>>>(partials, out5);
  return cudaGetLastError();
}

}  // namespace kkt
