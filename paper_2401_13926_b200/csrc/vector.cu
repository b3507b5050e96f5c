// Memory-bound vector kernels of the operator: SpMV (sparsecore.spmv, sparsecore.py:284-305)
// in the reference's accumulation order, and the fused residual statistics behind
// refine.nsr / nrbe / needs_refinement (refine.py:62-92).  blockIdx.y = system; vectors are
// system-major [nb][n].  Reductions use a fixed grid and a fixed-shape tree, so results are
// run-to-run deterministic.
#include <cuda_runtime.h>

#include "device.h"
#include "kernels.cuh"

namespace kkt {

// y = K x for one row in the reference order.  Symmetric-lower input: the reference sums
// the stored lower row (cols <= i, ascending) and, separately, the mirrored strict entries
// (rows k > i ascending) and adds the two bincounts; in the expanded general row these are
// the two halves split at the diagonal.
__device__ __forceinline__ double row_dot(const DevPlan &d, const double *__restrict__ av,
                                          const double *__restrict__ x, int i) {
  const int b = d.A_rp[i], s = d.A_split[i], e = d.A_rp[i + 1];
  const int *__restrict__ ci = d.A_ci;
  double s1 = 0.0, s2 = 0.0;
  for (int p0 = b; p0 < e; p0 += 8) {  // 8 independent loads in flight, then the ordered sum
    int c[8];
    double v[8], xv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (p0 + u < e) {
        c[u] = ci[p0 + u];
        v[u] = av[p0 + u];
      }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (p0 + u < e) xv[u] = x[c[u]];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (p0 + u < e) {
        const double t = __dmul_rn(v[u], xv[u]);
        if (d.sym_lower && p0 + u >= s) s2 = __dadd_rn(s2, t);
        else s1 = __dadd_rn(s1, t);
      }
  }
  return d.sym_lower ? __dadd_rn(s1, s2) : s1;
}

// The same row sums for the 32 rows r0 .. r0+31 of a warp (lane l: row r0 + l), with the
// tile's entries loaded coalesced (lanes over entries, 8 per lane in flight per 256-entry
// chunk) and their products staged in shared memory; each lane then adds its own row's
// products in entry order (the split as above), so every row is bitwise row_dot's.  The
// kernels keep the thread -> row mapping of the per-row loop (thread t of block b: rows
// 256 b + t + k * 256 * grid), so the norm partials are bitwise unchanged too.
constexpr int TILE_CHUNK = 256;
__device__ __forceinline__ double tile_dot(const DevPlan &d, const double *__restrict__ av,
                                           const double *__restrict__ x, int r0, int lane,
                                           double *__restrict__ prod) {
  const int *__restrict__ ci = d.A_ci;
  const int r = r0 + lane;
  const bool valid = r < d.n;
  const int rb = valid ? d.A_rp[r] : 0, re = valid ? d.A_rp[r + 1] : 0, rs = valid ? d.A_split[r] : 0;
  const int e0 = __shfl_sync(0xffffffffu, rb, 0);
  const int e1 = __shfl_sync(0xffffffffu, re, min(31, d.n - 1 - r0));
  double s1 = 0.0, s2 = 0.0;
  for (int c0 = e0; c0 < e1; c0 += TILE_CHUNK) {
    const int cn = min(TILE_CHUNK, e1 - c0);
    int c[8];
    double v[8], xv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int q = lane + 32 * u;
      if (q < cn) {
        c[u] = ci[c0 + q];
        v[u] = av[c0 + q];
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (lane + 32 * u < cn) xv[u] = x[c[u]];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (lane + 32 * u < cn) prod[lane + 32 * u] = __dmul_rn(v[u], xv[u]);
    __syncwarp();
    const int b = max(rb, c0), e = min(re, c0 + cn);
    for (int q = b; q < e; ++q) {
      const double t = prod[q - c0];
      if (d.sym_lower && q >= rs) s2 = __dadd_rn(s2, t);
      else s1 = __dadd_rn(s1, t);
    }
    __syncwarp();
  }
  return d.sym_lower ? __dadd_rn(s1, s2) : s1;
}

// out = K x, or out = bsub - K x; optional ||out||^2 block partials [nb][rb].
__global__ void __launch_bounds__(RED_THREADS) k_spmv(DevPlan d, const double *__restrict__ x,
                                                      double *__restrict__ out,
                                                      const double *__restrict__ bsub,
                                                      double *__restrict__ nrm_out) {
  __shared__ double sh[32];
  const int sys = blockIdx.y;
  if (!sys_active(d, sys)) return;
  const size_t off = (size_t)sys * d.n;
  const double *av = d.A_vals + (size_t)sys * d.nnz_a;
  x += off;
  out += off;
  if (bsub) bsub += off;
  __shared__ double prod_all[RED_THREADS / 32][TILE_CHUNK];
  double *prod = prod_all[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  double loc = 0.0;
  bool bad = false;
  for (int r0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31); r0 < d.n; r0 += gridDim.x * blockDim.x) {
    const int i = r0 + lane;
    const double y = tile_dot(d, av, x, r0, lane, prod);
    if (i < d.n) {
      if (!isfinite(y)) bad = true;
      const double o = bsub ? __dsub_rn(bsub[i], y) : y;
      out[i] = o;
      loc = __dadd_rn(loc, __dmul_rn(o, o));
    }
  }
  if (bad) atomicOr(&d.scal[(size_t)sys * SCAL_STRIDE + SC_NONFINITE], 1ull);
  if (nrm_out) {
    const double t = block_sum<RED_THREADS>(loc, sh);
    if (threadIdx.x == 0) nrm_out[(size_t)sys * gridDim.x + blockIdx.x] = t;
  }
}

// out[sys * ostride + v] = sum (or sqrt of the sum) of partials[sys][v][0..nblk), fixed order.
__global__ void k_reduce_partials(const double *__restrict__ partials, int nvec, int nblk,
                                  double *__restrict__ out, int ostride, int op_sqrt) {
  const int v = blockIdx.x, sys = blockIdx.y;
  const double *p = partials + ((size_t)sys * nvec + v) * nblk;
  double s = 0.0;
  for (int b = threadIdx.x; b < nblk; b += 32) s += p[b];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) out[(size_t)sys * ostride + v] = op_sqrt ? sqrt(s) : s;
}

// Residual statistics for (r, x): e = r - K x (spmv order), then per system
// {||e||_2^2, max|e|, ||x||_2^2, max|x|, ||r||_2^2} block partials [nb][5][rb].
__global__ void __launch_bounds__(RED_THREADS) k_resid_stats(DevPlan d, const double *__restrict__ r,
                                                             const double *__restrict__ x,
                                                             double *__restrict__ partials) {
  __shared__ double sh[32];
  const int sys = blockIdx.y, nblk = gridDim.x;
  const size_t off = (size_t)sys * d.n;
  const double *av = d.A_vals + (size_t)sys * d.nnz_a;
  r += off;
  x += off;
  double *part = partials + (size_t)sys * 5 * nblk;
  __shared__ double prod_all[RED_THREADS / 32][TILE_CHUNK];
  double *prod = prod_all[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  double e2 = 0.0, emax = 0.0, x2 = 0.0, xmax = 0.0, r2 = 0.0;
  for (int r0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31); r0 < d.n; r0 += gridDim.x * blockDim.x) {
    const int i = r0 + lane;
    const double y = tile_dot(d, av, x, r0, lane, prod);
    if (i < d.n) {
      const double ei = __dsub_rn(r[i], y);
      e2 += ei * ei;
      emax = fmax(emax, fabs(ei));
      x2 += x[i] * x[i];
      xmax = fmax(xmax, fabs(x[i]));
      r2 += r[i] * r[i];
    }
  }
  double t;
  t = block_sum<RED_THREADS>(e2, sh);
  if (threadIdx.x == 0) part[0 * nblk + blockIdx.x] = t;
  t = block_sum<RED_THREADS>(x2, sh);
  if (threadIdx.x == 0) part[2 * nblk + blockIdx.x] = t;
  t = block_sum<RED_THREADS>(r2, sh);
  if (threadIdx.x == 0) part[4 * nblk + blockIdx.x] = t;
  emax = warp_max(emax);
  xmax = warp_max(xmax);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = emax;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < RED_THREADS / 32; ++w) m = fmax(m, sh[w]);
    part[1 * nblk + blockIdx.x] = m;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = xmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < RED_THREADS / 32; ++w) m = fmax(m, sh[w]);
    part[3 * nblk + blockIdx.x] = m;
  }
}

// out[sys][5] = {||e||_2, ||e||_inf, ||x||_2, ||x||_inf, ||r||_2}
__global__ void k_resid_final(const double *__restrict__ partials, int nblk, double *__restrict__ out) {
  const int v = blockIdx.x, sys = blockIdx.y;
  const double *p = partials + ((size_t)sys * 5 + v) * nblk;
  double s = 0.0;
  const bool is_max = (v == 1 || v == 3);
  for (int b = threadIdx.x; b < nblk; b += 32) s = is_max ? fmax(s, p[b]) : s + p[b];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double q = __shfl_down_sync(0xffffffffu, s, o);
    s = is_max ? fmax(s, q) : s + q;
  }
  if (threadIdx.x == 0) out[(size_t)sys * 5 + v] = is_max ? s : sqrt(s);
}

cudaError_t launch_spmv(const DevPlan &d, const double *x, double *out, const double *bsub,
                        double *nrm_partials, cudaStream_t s) {
  k_spmv<<<dim3(d.rb, d.nb), RED_THREADS, 0, s>>>(d, x, out, bsub, nrm_partials);
  return cudaGetLastError();
}

cudaError_t launch_reduce_partials(const DevPlan &d, const double *partials, int nvec, double *out,
                                   int ostride, int op_sqrt, cudaStream_t s) {
  k_reduce_partials<<<dim3(nvec, d.nbp), 32, 0, s>>>(partials, nvec, d.rb, out, ostride, op_sqrt);
  return cudaGetLastError();
}

cudaError_t launch_resid_stats(const DevPlan &d, const double *r, const double *x,
                               double *partials, double *out5, cudaStream_t s) {
  k_resid_stats<<<dim3(d.rb, d.nb), RED_THREADS, 0, s>>>(d, r, x, partials);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_resid_final<<<dim3(5, d.nb), 32, 0, s>>>(partials, d.rb, out5);
  return cudaGetLastError();
}

}  // namespace kkt
