// B200 (sm_100a) device path: refactorization, triangular solves, SpMV, FGMRES(m)+CGS2 and
// the FGMRES iterative-refinement driver, behind the C ABI of include/kktb200.h.
//
// Reference behaviour reproduced (pkg/src/kktsolve/...):
//   k_expand_norms  sparsecore.to_general values (:263) + inf_norm (:333) + max|a|
//   k_refactor      direct_lu.refactorize (:297-356)        bitwise (ordered, non-FMA)
//   k_trsv<false>   direct_lu.lu_solve forward sweep (:369-371) bitwise (ascending j)
//   k_trsv<true>    direct_lu.lu_solve backward sweep (:372-377) bitwise (descending j)
//   k_spmv          sparsecore.spmv (:284-305)              bitwise (bincount order)
//   k_dots / k_cgs  krylov.cgs2_step (:93-105)              reassociated (tree sums)
//   k_givens        krylov.fgmres Hessenberg/Givens (:166-186), on device
//   k_solve_upper   krylov._solve_upper (:211-216)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "device.h"
#include "kernels.cuh"

namespace kkt {

constexpr int RED_BLOCKS = 296;  // fixed => reductions are run-to-run deterministic
constexpr int RED_THREADS = 256;
constexpr double HAPPY_BREAKDOWN_RTOL = 1e-14;  // krylov.py:25
constexpr double PATCH_RELATIVE_FLOOR = 1e-12;  // direct_lu.py:32

#define CUDA_TRY(expr)                                                                  \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      return set_error(_e == cudaErrorMemoryAllocation ? KKT_ERR_OOM : KKT_ERR_CUDA,     \
                       std::string(#expr) + ": " + cudaGetErrorString(_e));             \
  } while (0)

// ============================================================================
// Operator values: expand caller layout -> general CSR, inf-norms, max|a|.
// One thread per row; sums in entry order (np.bincount order => bitwise).
// ============================================================================
__global__ void k_expand_norms(DevPlan d) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.n) return;
  const int b = d.A_rp[i], s = d.A_split[i], e = d.A_rp[i + 1];
  double sg = 0.0, s1 = 0.0, s2 = 0.0, mx = 0.0;
  for (int p = b; p < e; ++p) {
    const double v = d.in_vals[d.sym_lower ? d.gen_src[p] : p];
    d.A_vals[p] = v;
    const double a = fabs(v);
    sg = __dadd_rn(sg, a);
    if (p < s) s1 = __dadd_rn(s1, a); else s2 = __dadd_rn(s2, a);
    mx = fmax(mx, a);
  }
  // refactorize uses inf_norm of the general matrix (direct_lu.py:318);
  // nsr/nrbe use inf_norm of the symmetric-lower operator (two bincounts, refine.py:70).
  atomic_max_nonneg(&d.scal[SC_MAXABS_A], mx);
  atomic_max_nonneg(&d.scal[SC_INFNORM], sg);
  const double op = d.sym_lower ? __dadd_rn(s1, s2) : sg;
  atomic_max_nonneg(&d.scal[SC_COUNT + 0], op);
}

// ============================================================================
// Refactorization: persistent warp-per-column, sync-free.
// Columns are dispatched in DAG-level order; a warp walks so(j) in the reference's
// topological order and waits on `done[k]` only for the column it needs next, so the
// critical path is the pipelined column walk, not the level-synchronous chain.
// Column j's pattern (U rows, diagonal, L rows; sorted positions) lives in shared memory;
// every update pair carries its precomputed slot (uint16).
// ============================================================================
__global__ void __launch_bounds__(256) k_refactor(DevPlan d, int *counter, int epoch) {
  // eps_patch = 1e-12 * inf_norm(Ag)                                 (direct_lu.py:318)
  const double eps = __dmul_rn(PATCH_RELATIVE_FLOOR, __longlong_as_double((long long)d.scal[SC_INFNORM]));
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  double *x = smem + (size_t)wib * d.maxpat;
  unsigned long long *patched_ctr = &d.scal[SC_PATCHED];
  while (true) {
    int idx = 0;
    if (lane == 0) idx = atomicAdd(counter, 1);
    idx = __shfl_sync(0xffffffffu, idx, 0);
    if (idx >= d.n) break;
    const int j = d.col_order[idx];
    const int ub = d.Up[j], nu = d.Up[j + 1] - ub;
    const int lb = d.Lp[j], nl = d.Lp[j + 1] - lb;
    const int np = nu + 1 + nl;
    for (int s = lane; s < np; s += 32) x[s] = 0.0;
    __syncwarp();
    // x[a_tgt] = avals[a_src]                                   (direct_lu.py:323)
    for (int q = d.ap_ptr[j] + lane; q < d.ap_ptr[j + 1]; q += 32) x[d.a_slot[q]] = d.A_vals[d.a_src[q]];
    __syncwarp();
    // for k in so(j): x[Li(k)] -= Lx(k) * x[k]                   (direct_lu.py:324-326)
    const int t_end = d.so_ptr[j + 1];
    for (int t0 = d.so_ptr[j]; t0 < t_end; t0 += 32) {
      const int t = t0 + lane;
      const bool valid = t < t_end;
      int my_k = 0, my_slot = 0, my_ub = 0, my_lb = 0, my_cnt = 0;
      if (valid) {
        my_k = d.so_data[t];
        my_slot = d.so_slot[t];
        my_ub = d.upd_ptr[t];
        my_lb = d.Lp[my_k];
        my_cnt = d.Lp[my_k + 1] - my_lb;
      }
      const int nsteps = min(32, t_end - t0);
      int ready_upto = 0;
      for (int i = 0; i < nsteps; ++i) {
        if (i >= ready_upto) {
          // poll until step i is ready; extend over the ready prefix of this chunk
          while (true) {
            const bool r = !valid || lane < i || ld_acquire(&d.done[my_k]) == epoch;
            const unsigned nr = __ballot_sync(0xffffffffu, !r);
            if (!(nr & (1u << i))) {
              ready_upto = nr ? (__ffs(nr) - 1) : 32;
              break;
            }
            __nanosleep(32);
          }
          __syncwarp();  // order the acquiring lanes' loads before everyone's L(:,k) reads
        }
        const int kslot = __shfl_sync(0xffffffffu, my_slot, i);
        const int ubase = __shfl_sync(0xffffffffu, my_ub, i);
        const int lbase = __shfl_sync(0xffffffffu, my_lb, i);
        const int cnt = __shfl_sync(0xffffffffu, my_cnt, i);
        const double xk = x[kslot];
        for (int e = lane; e < cnt; e += 32) {
          const int s = d.upd_slot[ubase + e];
          const double l = ldcg(&d.Lx[lbase + e]);
          x[s] = __dsub_rn(x[s], __dmul_rn(l, xk));
        }
        __syncwarp();
      }
    }
    // U(:,j) = x[Ui]; u_jj = x[j]; patch; L(:,j) = x[Li] / u_jj   (direct_lu.py:327-344)
    double gm = 0.0;
    for (int s = lane; s < nu; s += 32) {
      const double v = x[s];
      d.Ux[ub + s] = v;
      d.Uv[d.Umap[ub + s]] = v;
      gm = fmax(gm, fabs(v));
    }
    double ujj = x[nu];
    gm = fmax(gm, fabs(ujj));
    if (fabs(ujj) < eps) {
      ujj = (ujj >= 0.0) ? eps : -eps;
      if (lane == 0) atomicAdd(patched_ctr, 1ull);
    }
    for (int s = lane; s < nl; s += 32) {
      const double v = x[nu + 1 + s];
      gm = fmax(gm, fabs(v));
      const double l = __ddiv_rn(v, ujj);
      d.Lx[lb + s] = l;
      d.Lv[d.Lmap[lb + s]] = l;
    }
    gm = warp_max(gm);
    __syncwarp();
    if (lane == 0) {
      d.udiag[j] = ujj;
      atomic_max_nonneg(&d.scal[SC_GMAX], gm);
      __threadfence();
      st_release(&d.done[j], epoch);
    }
    __syncwarp();
  }
}

__global__ void k_diag_stats(DevPlan d) {
  double mx = 0.0, mn = INFINITY;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d.n; i += gridDim.x * blockDim.x) {
    const double a = fabs(d.udiag[i]);
    mx = fmax(mx, a);
    mn = fmin(mn, a);
  }
  atomic_max_nonneg(&d.scal[SC_MAXPIV], mx);
  if (mn < INFINITY) atomic_min_nonneg(&d.scal[SC_MINPIV], mn);
}

// ============================================================================
// Triangular solves: persistent, sync-free, warp per row, rows dispatched round-robin in
// level order (deadlock-free because every warp of the grid is resident).  Each row
// accumulates its entries strictly in the reference order (ascending j for L, descending j
// for U), products and differences rounded separately => bitwise equal to lu_solve.
// Readiness: per-row flag == epoch (release/acquire).  U runs in place on y like :372-375.
// ============================================================================
template <bool IS_U>
__global__ void __launch_bounds__(256) k_trsv(DevPlan d, const double *__restrict__ b,
                                              double *__restrict__ xout, int epoch) {
  const int lane = threadIdx.x & 31;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int *order = IS_U ? d.U_order : d.L_order;
  const int *rp = IS_U ? d.Urp : d.Lrp;
  const int *ci = IS_U ? d.Uci : d.Lci;
  const double *vals = IS_U ? d.Uv : d.Lv;
  bool bad = false;
  for (int idx = gwarp; idx < d.n; idx += nwarps) {
    const int r = order[idx];
    double acc = IS_U ? ldcg(&d.y[r]) : b[d.row_perm[r]];
    const int beg = rp[r], end = rp[r + 1];
    for (int c0 = beg; c0 < end; c0 += 32) {
      const int e = c0 + lane;
      double p = 0.0;
      if (e < end) {
        const int col = ci[e];
        const double v = vals[e];
        while (ld_acquire(&d.tflag[col]) != epoch) {
        }
        p = __dmul_rn(v, ldcg(&d.y[col]));
      }
      const int cnt = min(32, end - c0);
      for (int i = 0; i < cnt; ++i) acc = __dsub_rn(acc, __shfl_sync(0xffffffffu, p, i));
    }
    if (lane == 0) {
      double w = acc;
      if (IS_U) {
        w = __ddiv_rn(acc, d.udiag[r]);
        xout[d.col_perm[r]] = w;
        if (!isfinite(w)) bad = true;
      }
      __stcg(&d.y[r], w);
      st_release(&d.tflag[r], epoch);
    }
  }
  if (IS_U && bad) atomicOr((unsigned long long *)&d.scal[SC_NONFINITE], 1ull);
}

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
  if (bad) atomicOr((unsigned long long *)&d.scal[SC_NONFINITE], 1ull);
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

// ============================================================================
// FGMRES(m) with CGS2 (krylov.py:117-208).
// ============================================================================
struct KState {
  double beta0, beta, target, floor, est, hj1;
  int j, stop, converged, pad;
};

struct Krylov {
  int m = 0, n = 0;
  double *V = nullptr;  // (m+1) x n
  double *Z = nullptr;  // m x n
  double *w = nullptr, *w1 = nullptr, *r = nullptr, *x = nullptr;
  double *sr = nullptr, *sx0 = nullptr, *sx = nullptr;  // kkt_dev_step staging
  double *h1 = nullptr, *h2 = nullptr, *H = nullptr, *cs = nullptr, *sn = nullptr, *g = nullptr,
         *yv = nullptr, *nrm = nullptr, *beta = nullptr;
  KState *st = nullptr;
  double *partials = nullptr;  // (m+1) * RED_BLOCKS
  void *mem = nullptr;
};

// h[i] = V_i . w for i < nvec, block partials (vectors in groups of 8, w re-read from L2).
__global__ void __launch_bounds__(RED_THREADS) k_dots(const double *__restrict__ V, int nvec, int n,
                                                      const double *__restrict__ w,
                                                      double *__restrict__ partials) {
  __shared__ double sh[32];
  for (int g0 = 0; g0 < nvec; g0 += 8) {
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int gn = min(8, nvec - g0);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
      const double wi = w[i];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < gn) acc[q] += V[(size_t)(g0 + q) * n + i] * wi;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (q < gn) {
        const double t = block_sum<RED_THREADS>(acc[q], sh);
        if (threadIdx.x == 0) partials[(size_t)(g0 + q) * RED_BLOCKS + blockIdx.x] = t;
      }
    }
  }
}

// w_out = w_in - sum_i V_i h[i] (sequential i); then either dots V.w_out (mode 0) or
// ||w_out||^2 (mode 1) as block partials.
__global__ void __launch_bounds__(RED_THREADS) k_cgs(const double *__restrict__ V, int nvec, int n,
                                                     const double *__restrict__ w_in,
                                                     const double *__restrict__ h,
                                                     double *__restrict__ w_out, int mode,
                                                     double *__restrict__ partials) {
  __shared__ double sh[32];
  __shared__ double hs[64];
  for (int q = threadIdx.x; q < nvec; q += blockDim.x) hs[q] = h[q];
  __syncthreads();
  if (mode == 1) {
    double acc = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
      double t = 0.0;
      for (int q = 0; q < nvec; ++q) t += V[(size_t)q * n + i] * hs[q];
      const double o = w_in[i] - t;
      w_out[i] = o;
      acc += o * o;
    }
    const double t = block_sum<RED_THREADS>(acc, sh);
    if (threadIdx.x == 0) partials[blockIdx.x] = t;
    return;
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double t = 0.0;
    for (int q = 0; q < nvec; ++q) t += V[(size_t)q * n + i] * hs[q];
    w_out[i] = w_in[i] - t;
  }
}

// Hessenberg column j, Givens rotations, residual estimate (krylov.py:166-186).
__global__ void k_givens(KState *st, int j, int m, const double *__restrict__ h1,
                         const double *__restrict__ h2, const double *__restrict__ nrm2,
                         double *H, double *cs, double *sn, double *g, double *status) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  // H is (m+1) x m row-major: H[i*m + j]
  for (int i = 0; i <= j; ++i) H[i * m + j] = h1[i] + h2[i];
  const double hj1 = sqrt(nrm2[0]);
  H[(j + 1) * m + j] = hj1;
  for (int i = 0; i < j; ++i) {
    const double a = H[i * m + j], b = H[(i + 1) * m + j];
    const double t = __dadd_rn(__dmul_rn(cs[i], a), __dmul_rn(sn[i], b));
    H[(i + 1) * m + j] = __dadd_rn(__dmul_rn(-sn[i], a), __dmul_rn(cs[i], b));
    H[i * m + j] = t;
  }
  const double denom = hypot(H[j * m + j], H[(j + 1) * m + j]);
  cs[j] = __ddiv_rn(H[j * m + j], denom);
  sn[j] = __ddiv_rn(H[(j + 1) * m + j], denom);
  H[j * m + j] = denom;
  H[(j + 1) * m + j] = 0.0;
  g[j + 1] = __dmul_rn(-sn[j], g[j]);
  g[j] = __dmul_rn(cs[j], g[j]);
  const double est = fabs(g[j + 1]);
  st->est = est;
  st->hj1 = hj1;
  st->j = j;
  const int stop = (est <= st->target || hj1 <= st->floor) ? 1 : 0;
  st->stop = stop;
  status[0] = est;
  status[1] = stop;
  status[2] = hj1;
}

__global__ void k_scale(const double *__restrict__ in, double *__restrict__ out, int n,
                        const double *__restrict__ den) {
  const double dv = den[0];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = __ddiv_rn(in[i], dv);
}

__global__ void k_cycle_init(double *g, int m, const double *beta, double *H) {
  for (int i = threadIdx.x; i <= m; i += blockDim.x) g[i] = (i == 0) ? beta[0] : 0.0;
  for (int i = threadIdx.x; i < (m + 1) * m; i += blockDim.x) H[i] = 0.0;
}

// y = R^{-1} g on the leading k x k block (krylov.py:211-216).
__global__ void k_solve_upper(const double *H, int m, const double *g, int k, double *y) {
  if (threadIdx.x != 0) return;
  for (int i = k - 1; i >= 0; --i) {
    double dot = 0.0;
    for (int q = i + 1; q < k; ++q) dot = __dadd_rn(dot, __dmul_rn(H[i * m + q], y[q]));
    y[i] = __ddiv_rn(__dsub_rn(g[i], dot), H[i * m + i]);
  }
}

// x = x + (sum_q Z_q y_q)   (krylov.py:190: the matvec first, then the add)
__global__ void k_update_x(double *__restrict__ x, const double *__restrict__ Z, int n,
                           const double *__restrict__ y, int k) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double t = 0.0;
    for (int q = 0; q < k; ++q) t = __dadd_rn(t, __dmul_rn(Z[(size_t)q * n + i], y[q]));
    x[i] = __dadd_rn(x[i], t);
  }
}

// ============================================================================
// Host-side orchestration
// ============================================================================
static size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

template <typename T>
static T *carve(char *&cur, size_t count) {
  T *p = reinterpret_cast<T *>(cur);
  cur += align_up(count * sizeof(T) + 1);
  return p;
}

template <typename S, typename T>
static std::vector<T> narrow(const std::vector<S> &v) {
  std::vector<T> o(v.size());
  for (size_t i = 0; i < v.size(); ++i) o[i] = (T)v[i];
  return o;
}

static std::vector<int> to_i32(const std::vector<int64_t> &v) { return narrow<int64_t, int>(v); }

static int upload(void *dst, const void *src, size_t bytes, cudaStream_t s) {
  if (!bytes) return KKT_OK;
  CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
  return KKT_OK;
}

#define UP(dst, vec) \
  if ((rc = upload(dst, vec.data(), vec.size() * sizeof(vec[0]), dev->stream)) != KKT_OK) return rc

static int alloc_krylov(Device *dev, int m) {
  Krylov *K = new Krylov();
  K->m = m;
  K->n = dev->d.n;
  const size_t n = (size_t)dev->d.n;
  size_t bytes = 0;
  bytes += align_up(8 * (m + 1) * n + 1) + align_up(8 * m * n + 1) + 7 * align_up(8 * n + 1);
  bytes += 2 * align_up(8 * (m + 1) + 1) + align_up(8 * (m + 1) * m + 1) + 4 * align_up(8 * (m + 1) + 1);
  bytes += 2 * align_up(64) + align_up(sizeof(KState)) + align_up(8 * (m + 2) * RED_BLOCKS + 1);
  cudaError_t e = cudaMalloc(&K->mem, bytes);
  if (e != cudaSuccess) {
    delete K;
    return set_error(KKT_ERR_OOM, "cudaMalloc of the FGMRES workspace failed");
  }
  char *cur = (char *)K->mem;
  K->V = carve<double>(cur, (m + 1) * n);
  K->Z = carve<double>(cur, (size_t)m * n);
  K->w = carve<double>(cur, n);
  K->w1 = carve<double>(cur, n);
  K->r = carve<double>(cur, n);
  K->x = carve<double>(cur, n);
  K->sr = carve<double>(cur, n);
  K->sx0 = carve<double>(cur, n);
  K->sx = carve<double>(cur, n);
  K->h1 = carve<double>(cur, m + 1);
  K->h2 = carve<double>(cur, m + 1);
  K->H = carve<double>(cur, (size_t)(m + 1) * m);
  K->cs = carve<double>(cur, m + 1);
  K->sn = carve<double>(cur, m + 1);
  K->g = carve<double>(cur, m + 1);
  K->yv = carve<double>(cur, m + 1);
  K->nrm = carve<double>(cur, 8);
  K->beta = carve<double>(cur, 8);
  K->st = carve<KState>(cur, 1);
  K->partials = carve<double>(cur, (size_t)(m + 2) * RED_BLOCKS);
  if (dev->kry) {
    cudaFree(dev->kry->mem);
    delete dev->kry;
  }
  dev->kry = K;
  return KKT_OK;
}

static int create(const Symbolic &S, const int64_t *A_rp, const int64_t *A_ci, int64_t in_nnz,
                  const int64_t *gen_src, const kkt_device_opts *opts, Device *&out) {
  out = nullptr;
  Device *dev = new Device();
  int rc = build_plan(S, A_rp, A_ci, in_nnz, gen_src, dev->h);
  if (rc != KKT_OK) {
    delete dev;
    return rc;
  }
  const HostPlan &h = dev->h;
  dev->device = opts ? opts->device : 0;
  dev->restart_m = (opts && opts->restart_m > 0) ? opts->restart_m : 10;
  if (opts && opts->batch > 1) {
    delete dev;
    return set_error(KKT_ERR_BAD_ARG, "batch > 1 is not supported by this handle type");
  }
  cudaError_t ce = cudaSetDevice(dev->device);
  if (ce != cudaSuccess) {
    delete dev;
    return set_error(KKT_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(ce));
  }
  cudaDeviceGetAttribute(&dev->sm_count, cudaDevAttrMultiProcessorCount, dev->device);
  ce = cudaStreamCreateWithFlags(&dev->stream, cudaStreamNonBlocking);
  if (ce != cudaSuccess) {
    delete dev;
    return set_error(KKT_ERR_CUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(ce));
  }
  DevPlan &d = dev->d;
  d.n = h.n;
  d.sym_lower = 0;
  d.has_lower = h.has_lower;
  d.nnz_a = h.nnz_a;
  d.in_nnz = h.in_nnz;
  d.nnz_L = h.nnz_L;
  d.nnz_U = h.nnz_U;
  d.n_so = (int64_t)h.so_data.size();
  d.n_upd = (int64_t)h.upd_slot.size();
  d.n_ap = (int64_t)h.a_src.size();
  d.maxpat = h.maxpat;
  const size_t n = (size_t)h.n;
  size_t bytes = 0;
  auto acc = [&](size_t b) { bytes += align_up(b + 1); };
  acc(4 * (n + 1)); acc(4 * d.nnz_a); acc(4 * n); acc(4 * d.nnz_a);            // A_rp ci split gen_src
  acc(8 * std::max(d.in_nnz, d.nnz_a)); acc(8 * d.nnz_a);                                         // in_vals A_vals
  acc(4 * (n + 1)); acc(4 * d.n_so); acc(4 * (d.n_so + 1)); acc(4 * (n + 1));  // so_ptr so_data upd_ptr ap_ptr
  acc(4 * d.n_ap); acc(4 * n); acc(4 * (n + 1)); acc(4 * (n + 1));             // a_src col_order Lp Up
  acc(4 * d.nnz_L); acc(4 * d.nnz_U);                                          // Lmap Umap
  acc(2 * d.n_so); acc(2 * d.n_upd); acc(2 * d.n_ap);                          // slots
  acc(8 * d.nnz_L); acc(8 * d.nnz_U); acc(8 * n); acc(4 * n);                  // Lx Ux udiag done
  acc(4 * (n + 1)); acc(4 * d.nnz_L); acc(4 * (n + 1)); acc(4 * d.nnz_U);      // Lrp Lci Urp Uci
  acc(4 * n); acc(4 * n); acc(4 * n); acc(4 * n);                              // orders, perms
  acc(8 * d.nnz_L); acc(8 * d.nnz_U); acc(4 * n); acc(8 * n);                  // Lv Uv tflag y
  acc(8 * 32); acc(64); acc(8 * 8 * RED_BLOCKS);                               // scal ticket partials
  ce = cudaMalloc(&dev->arena, bytes);
  if (ce != cudaSuccess) {
    cudaStreamDestroy(dev->stream);
    delete dev;
    return set_error(KKT_ERR_OOM, "cudaMalloc of the device plan failed");
  }
  dev->arena_bytes = bytes;
  char *cur = (char *)dev->arena;
  d.A_rp = carve<int>(cur, n + 1);
  d.A_ci = carve<int>(cur, d.nnz_a);
  d.A_split = carve<int>(cur, n);
  d.gen_src = carve<int>(cur, d.nnz_a);
  d.in_vals = carve<double>(cur, std::max(d.in_nnz, d.nnz_a));
  d.A_vals = carve<double>(cur, d.nnz_a);
  d.so_ptr = carve<int>(cur, n + 1);
  d.so_data = carve<int>(cur, d.n_so);
  d.upd_ptr = carve<int>(cur, d.n_so + 1);
  d.ap_ptr = carve<int>(cur, n + 1);
  d.a_src = carve<int>(cur, d.n_ap);
  d.col_order = carve<int>(cur, n);
  d.Lp = carve<int>(cur, n + 1);
  d.Up = carve<int>(cur, n + 1);
  d.Lmap = carve<int>(cur, d.nnz_L);
  d.Umap = carve<int>(cur, d.nnz_U);
  d.so_slot = carve<uint16_t>(cur, d.n_so);
  d.upd_slot = carve<uint16_t>(cur, d.n_upd);
  d.a_slot = carve<uint16_t>(cur, d.n_ap);
  d.Lx = carve<double>(cur, d.nnz_L);
  d.Ux = carve<double>(cur, d.nnz_U);
  d.udiag = carve<double>(cur, n);
  d.done = carve<int>(cur, n);
  d.Lrp = carve<int>(cur, n + 1);
  d.Lci = carve<int>(cur, d.nnz_L);
  d.Urp = carve<int>(cur, n + 1);
  d.Uci = carve<int>(cur, d.nnz_U);
  d.L_order = carve<int>(cur, n);
  d.U_order = carve<int>(cur, n);
  d.row_perm = carve<int>(cur, n);
  d.col_perm = carve<int>(cur, n);
  d.Lv = carve<double>(cur, d.nnz_L);
  d.Uv = carve<double>(cur, d.nnz_U);
  d.tflag = carve<int>(cur, n);
  d.y = carve<double>(cur, n);
  d.scal = carve<unsigned long long>(cur, 32);
  d.ticket = carve<int>(cur, 16);
  d.partials = carve<double>(cur, 8 * RED_BLOCKS);
  dev->d = d;
  // upload
  UP(d.A_rp, to_i32(h.A_rp));
  UP(d.A_ci, to_i32(h.A_ci));
  UP(d.A_split, to_i32(h.A_split));
  UP(d.gen_src, to_i32(h.gen_src));
  UP(d.so_ptr, to_i32(h.so_ptr));
  UP(d.so_data, h.so_data);
  UP(d.upd_ptr, h.upd_ptr);
  UP(d.ap_ptr, to_i32(h.ap_ptr));
  UP(d.a_src, h.a_src);
  UP(d.col_order, h.col_order);
  UP(d.Lp, to_i32(h.Lp));
  UP(d.Up, to_i32(h.Up));
  UP(d.Lmap, h.Lmap);
  UP(d.Umap, h.Umap);
  UP(d.so_slot, h.so_slot);
  UP(d.upd_slot, h.upd_slot);
  UP(d.a_slot, h.a_slot);
  UP(d.Lrp, h.Lrp);
  UP(d.Lci, h.Lci);
  UP(d.Urp, h.Urp);
  UP(d.Uci, h.Uci);
  UP(d.L_order, h.L_order);
  UP(d.U_order, h.U_order);
  UP(d.row_perm, to_i32(h.row_perm));
  UP(d.col_perm, to_i32(h.col_perm));
  // first factorization's values (so solve() works before any refactor, like LuFactors)
  UP(d.Lx, h.Lx0);
  UP(d.Ux, h.Ux0);
  UP(d.udiag, h.Udiag0);
  {
    std::vector<double> lv(h.nnz_L), uv(h.nnz_U);
    for (int64_t p = 0; p < h.nnz_L; ++p) lv[h.Lmap[p]] = h.Lx0[p];
    for (int64_t p = 0; p < h.nnz_U; ++p) uv[h.Umap[p]] = h.Ux0[p];
    UP(d.Lv, lv);
    UP(d.Uv, uv);
    CUDA_TRY(cudaStreamSynchronize(dev->stream));
  }
  CUDA_TRY(cudaMemsetAsync(d.done, 0, 4 * n, dev->stream));
  CUDA_TRY(cudaMemsetAsync(d.tflag, 0, 4 * n, dev->stream));
  CUDA_TRY(cudaMemsetAsync(d.scal, 0, 8 * 32, dev->stream));
  CUDA_TRY(cudaMemsetAsync(d.ticket, 0, 64, dev->stream));
  // launch shapes
  dev->refactor_warps = 8;
  dev->refactor_smem = (size_t)dev->refactor_warps * d.maxpat * sizeof(double);
  while (dev->refactor_smem > 200 * 1024 && dev->refactor_warps > 1) {
    dev->refactor_warps /= 2;
    dev->refactor_smem = (size_t)dev->refactor_warps * d.maxpat * sizeof(double);
  }
  if (dev->refactor_smem > 220 * 1024) {
    cudaFree(dev->arena);
    cudaStreamDestroy(dev->stream);
    delete dev;
    return set_error(KKT_ERR_BAD_SHAPE, "column pattern too large for the shared-memory workspace");
  }
  CUDA_TRY(cudaFuncSetAttribute(k_refactor, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)std::max<size_t>(dev->refactor_smem, 48 * 1024)));
  int bps = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_refactor, 32 * dev->refactor_warps,
                                                         dev->refactor_smem));
  dev->refactor_blocks = std::max(1, bps) * dev->sm_count;
  int tb = 0, tb2 = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tb, k_trsv<false>, 256, 0));
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tb2, k_trsv<true>, 256, 0));
  dev->trsv_blocks = std::max(1, std::min(tb, tb2)) * dev->sm_count;
  CUDA_TRY(cudaMallocHost(&dev->pinned, 4096));
  rc = alloc_krylov(dev, dev->restart_m);
  if (rc != KKT_OK) return rc;
  CUDA_TRY(cudaStreamSynchronize(dev->stream));
  out = dev;
  return KKT_OK;
}

static void destroy(Device *dev) {
  if (!dev) return;
  cudaSetDevice(dev->device);
  if (dev->stream) cudaStreamSynchronize(dev->stream);
  if (dev->kry) {
    cudaFree(dev->kry->mem);
    delete dev->kry;
  }
  if (dev->arena) cudaFree(dev->arena);
  if (dev->pinned) cudaFreeHost(dev->pinned);
  if (dev->stream) cudaStreamDestroy(dev->stream);
  delete dev;
}

static int check_launch(Device *dev) {
  dev->launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(KKT_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(e));
  return KKT_OK;
}

#define LAUNCH_CHECK()                                   \
  do {                                                   \
    int _rc = check_launch(dev);                         \
    if (_rc != KKT_OK) return _rc;                       \
  } while (0)

static int set_values(Device *dev, const double *vals, int layout, int on_device) {
  DevPlan &d = dev->d;
  if (layout == KKT_LAYOUT_SYMMETRIC_LOWER && !d.has_lower)
    return set_error(KKT_ERR_BAD_ARG, "handle was created without the symmetric-lower map");
  if (layout != KKT_LAYOUT_GENERAL && layout != KKT_LAYOUT_SYMMETRIC_LOWER)
    return set_error(KKT_ERR_BAD_ARG, "unknown value layout");
  d.sym_lower = layout == KKT_LAYOUT_SYMMETRIC_LOWER ? 1 : 0;
  const int64_t cnt = d.sym_lower ? d.in_nnz : d.nnz_a;
  CUDA_TRY(cudaMemcpyAsync(d.in_vals, vals, 8 * (size_t)cnt,
                           on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, dev->stream));
  CUDA_TRY(cudaMemsetAsync(d.scal, 0, 8 * SC_MINPIV, dev->stream));
  CUDA_TRY(cudaMemsetAsync(&d.scal[SC_COUNT], 0, 8, dev->stream));
  k_expand_norms<<<(d.n + 255) / 256, 256, 0, dev->stream>>>(d);
  LAUNCH_CHECK();
  return KKT_OK;
}

static int refactor(Device *dev, const double *vals, int layout, int on_device, double *diag_out) {
  DevPlan &d = dev->d;
  int rc = set_values(dev, vals, layout, on_device);
  if (rc != KKT_OK) return rc;
  dev->epoch_refactor++;
  CUDA_TRY(cudaMemsetAsync(d.ticket, 0, 4, dev->stream));
  const unsigned long long big = 0x7FF0000000000000ull;  // +inf bits for the min
  CUDA_TRY(cudaMemcpyAsync(&d.scal[SC_MINPIV], &big, 8, cudaMemcpyHostToDevice, dev->stream));
  k_refactor<<<dev->refactor_blocks, 32 * dev->refactor_warps, dev->refactor_smem, dev->stream>>>(
      d, d.ticket, dev->epoch_refactor);
  LAUNCH_CHECK();
  k_diag_stats<<<dev->sm_count, 256, 0, dev->stream>>>(d);
  LAUNCH_CHECK();
  if (diag_out) {
    CUDA_TRY(cudaMemcpyAsync(dev->pinned, d.scal, 8 * SC_COUNT, cudaMemcpyDeviceToHost, dev->stream));
    CUDA_TRY(cudaStreamSynchronize(dev->stream));
    unsigned long long s[SC_COUNT];
    std::memcpy(s, dev->pinned, sizeof s);
    double v[SC_COUNT];
    std::memcpy(v, s, sizeof v);
    diag_out[0] = v[SC_MAXPIV];
    diag_out[1] = (d.n ? v[SC_MINPIV] : 0.0);
    diag_out[2] = (double)s[SC_PATCHED];
    diag_out[3] = v[SC_MAXABS_A] > 0 ? v[SC_GMAX] / v[SC_MAXABS_A] : 0.0;
  }
  return KKT_OK;
}

static int solve(Device *dev, const double *b, double *x) {
  DevPlan &d = dev->d;
  if (d.n == 0) return KKT_OK;
  dev->epoch_trsv++;
  k_trsv<false><<<dev->trsv_blocks, 256, 0, dev->stream>>>(d, b, x, dev->epoch_trsv);
  LAUNCH_CHECK();
  dev->epoch_trsv++;
  k_trsv<true><<<dev->trsv_blocks, 256, 0, dev->stream>>>(d, b, x, dev->epoch_trsv);
  LAUNCH_CHECK();
  return KKT_OK;
}

static int spmv(Device *dev, const double *x, double *y, const double *bsub, double *nrm_partials) {
  DevPlan &d = dev->d;
  k_spmv<<<RED_BLOCKS, RED_THREADS, 0, dev->stream>>>(d, x, y, bsub, nrm_partials);
  LAUNCH_CHECK();
  return KKT_OK;
}

static int residual_norms(Device *dev, const double *r, const double *x, double *out6) {
  DevPlan &d = dev->d;
  k_resid_stats<<<RED_BLOCKS, RED_THREADS, 0, dev->stream>>>(d, r, x, d.partials);
  LAUNCH_CHECK();
  k_resid_final<<<5, 32, 0, dev->stream>>>(d.partials, d.partials + 6 * RED_BLOCKS);
  LAUNCH_CHECK();
  CUDA_TRY(cudaMemcpyAsync(dev->pinned, d.partials + 6 * RED_BLOCKS, 5 * 8, cudaMemcpyDeviceToHost,
                           dev->stream));
  CUDA_TRY(cudaMemcpyAsync(dev->pinned + 5, &d.scal[SC_COUNT], 8, cudaMemcpyDeviceToHost, dev->stream));
  CUDA_TRY(cudaStreamSynchronize(dev->stream));
  std::memcpy(out6, dev->pinned, 6 * 8);
  return KKT_OK;
}

// krylov.fgmres with K = operator values and M = lu_solve (krylov.py:117-208).
static int fgmres(Device *dev, const double *b, const double *x0, double *xout, const kkt_krylov_cfg *cfg,
                  kkt_krylov_report *rep, double *hist, int hist_cap) {
  DevPlan &d = dev->d;
  const int n = d.n;
  if (cfg->m < 1) return set_error(KKT_ERR_BAD_ARG, "restart length m must be >= 1");
  if (!(cfg->tol > 0)) return set_error(KKT_ERR_BAD_ARG, "tol must be positive");
  if (cfg->m > 62) return set_error(KKT_ERR_BAD_ARG, "restart length m must be <= 62");
  if (!dev->kry || dev->kry->m < cfg->m) {
    int rc = alloc_krylov(dev, cfg->m);
    if (rc != KKT_OK) return rc;
  }
  Krylov &K = *dev->kry;
  const int m = cfg->m;
  std::memset(rep, 0, sizeof *rep);
  int hn = 0;
  auto push_hist = [&](double v) {
    if (hist && hn < hist_cap) hist[hn] = v;
    hn++;
  };
  CUDA_TRY(cudaMemsetAsync(&d.scal[SC_NONFINITE], 0, 8, dev->stream));
  CUDA_TRY(cudaMemcpyAsync(K.x, x0, 8 * (size_t)n, cudaMemcpyDeviceToDevice, dev->stream));
  // r = b - K x ; beta0
  int rc = spmv(dev, K.x, K.r, b, K.partials);
  if (rc) return rc;
  k_reduce_partials<<<1, 32, 0, dev->stream>>>(K.partials, 1, RED_BLOCKS, K.beta, 1);
  LAUNCH_CHECK();
  CUDA_TRY(cudaMemcpyAsync(dev->pinned, K.beta, 8, cudaMemcpyDeviceToHost, dev->stream));
  CUDA_TRY(cudaMemcpyAsync(dev->pinned + 1, &d.scal[SC_NONFINITE], 8, cudaMemcpyDeviceToHost, dev->stream));
  CUDA_TRY(cudaStreamSynchronize(dev->stream));
  if (((unsigned long long *)dev->pinned)[1]) {
    rep->nonfinite = 1;
    return set_error(KKT_ERR_NONFINITE, "operator produced a non-finite entry");
  }
  const double beta0 = dev->pinned[0];
  push_hist(beta0);
  rep->beta0 = beta0;
  if (beta0 == 0.0) {
    CUDA_TRY(cudaMemcpyAsync(xout, K.x, 8 * (size_t)n, cudaMemcpyDeviceToDevice, dev->stream));
    rep->converged = 1;
    rep->est_final = beta0;
    rep->true_final = 0.0;
    return KKT_OK;
  }
  KState st{};
  st.beta0 = beta0;
  st.target = cfg->tol * beta0;
  st.floor = HAPPY_BREAKDOWN_RTOL * beta0;
  CUDA_TRY(cudaMemcpyAsync(K.st, &st, sizeof st, cudaMemcpyHostToDevice, dev->stream));
  double beta = beta0, est = beta0;
  int converged = 0, iters = 0, restarts = 0;
  const int grid = RED_BLOCKS;
  for (int outer = 0; outer < cfg->max_outer; ++outer) {
    if (beta <= st.target) {
      converged = 1;
      break;
    }
    k_scale<<<grid, RED_THREADS, 0, dev->stream>>>(K.r, K.V, n, K.beta);  // V0 = r / beta
    LAUNCH_CHECK();
    k_cycle_init<<<1, 128, 0, dev->stream>>>(K.g, m, K.beta, K.H);
    LAUNCH_CHECK();
    int j_used = 0;
    bool stop = false;
    for (int j = 0; j < m; ++j) {
      double *Vj = K.V + (size_t)j * n;
      double *Zj = K.Z + (size_t)j * n;
      rc = solve(dev, Vj, Zj);  // z = M(V_j)
      if (rc) return rc;
      rc = spmv(dev, Zj, K.w, nullptr, nullptr);  // w = K z
      if (rc) return rc;
      const int nv = j + 1;
      k_dots<<<grid, RED_THREADS, 0, dev->stream>>>(K.V, nv, n, K.w, K.partials);
      LAUNCH_CHECK();
      k_reduce_partials<<<nv, 32, 0, dev->stream>>>(K.partials, nv, RED_BLOCKS, K.h1, 0);
      LAUNCH_CHECK();
      k_cgs<<<grid, RED_THREADS, 0, dev->stream>>>(K.V, nv, n, K.w, K.h1, K.w1, 0, nullptr);
      LAUNCH_CHECK();
      k_dots<<<grid, RED_THREADS, 0, dev->stream>>>(K.V, nv, n, K.w1, K.partials);
      LAUNCH_CHECK();
      k_reduce_partials<<<nv, 32, 0, dev->stream>>>(K.partials, nv, RED_BLOCKS, K.h2, 0);
      LAUNCH_CHECK();
      k_cgs<<<grid, RED_THREADS, 0, dev->stream>>>(K.V, nv, n, K.w1, K.h2, K.w, 1, K.partials);
      LAUNCH_CHECK();
      k_reduce_partials<<<1, 32, 0, dev->stream>>>(K.partials, 1, RED_BLOCKS, K.nrm, 0);
      LAUNCH_CHECK();
      k_givens<<<1, 32, 0, dev->stream>>>(K.st, j, m, K.h1, K.h2, K.nrm, K.H, K.cs, K.sn, K.g,
                                          K.partials + (size_t)(m + 1) * RED_BLOCKS);
      LAUNCH_CHECK();
      CUDA_TRY(cudaMemcpyAsync(dev->pinned, K.partials + (size_t)(m + 1) * RED_BLOCKS, 24,
                               cudaMemcpyDeviceToHost, dev->stream));
      CUDA_TRY(cudaMemcpyAsync(dev->pinned + 3, &d.scal[SC_NONFINITE], 8, cudaMemcpyDeviceToHost,
                               dev->stream));
      CUDA_TRY(cudaStreamSynchronize(dev->stream));
      if (((unsigned long long *)dev->pinned)[3]) {
        rep->nonfinite = 1;
        rep->iterations = iters;
        return set_error(KKT_ERR_NONFINITE, "preconditioner or operator produced a non-finite entry");
      }
      est = dev->pinned[0];
      stop = dev->pinned[1] != 0.0;
      push_hist(est);
      iters++;
      j_used = j + 1;
      if (stop) break;
      // V_{j+1} = w / hj1 (w holds w2 after the second CGS pass)
      k_scale<<<grid, RED_THREADS, 0, dev->stream>>>(K.w, K.V + (size_t)(j + 1) * n, n,
                                                      K.partials + (size_t)(m + 1) * RED_BLOCKS + 2);
      LAUNCH_CHECK();
    }
    k_solve_upper<<<1, 32, 0, dev->stream>>>(K.H, m, K.g, j_used, K.yv);
    LAUNCH_CHECK();
    k_update_x<<<grid, RED_THREADS, 0, dev->stream>>>(K.x, K.Z, n, K.yv, j_used);
    LAUNCH_CHECK();
    rc = spmv(dev, K.x, K.r, b, K.partials);  // r = b - K x
    if (rc) return rc;
    k_reduce_partials<<<1, 32, 0, dev->stream>>>(K.partials, 1, RED_BLOCKS, K.beta, 1);
    LAUNCH_CHECK();
    CUDA_TRY(cudaMemcpyAsync(dev->pinned, K.beta, 8, cudaMemcpyDeviceToHost, dev->stream));
    CUDA_TRY(cudaMemcpyAsync(dev->pinned + 1, &d.scal[SC_NONFINITE], 8, cudaMemcpyDeviceToHost,
                             dev->stream));
    CUDA_TRY(cudaStreamSynchronize(dev->stream));
    if (((unsigned long long *)dev->pinned)[1]) {
      rep->nonfinite = 1;
      return set_error(KKT_ERR_NONFINITE, "operator produced a non-finite entry");
    }
    beta = dev->pinned[0];
    restarts++;
    if (stop) {
      converged = 1;
      break;
    }
    if (beta <= st.target) {
      converged = 1;
      break;
    }
  }
  CUDA_TRY(cudaMemcpyAsync(xout, K.x, 8 * (size_t)n, cudaMemcpyDeviceToDevice, dev->stream));
  rep->iterations = iters;
  rep->precond_applications = iters;
  rep->converged = converged;
  rep->restarts = restarts;
  rep->est_final = est;
  rep->true_final = beta;
  return KKT_OK;
}

// ---------------------------------------------------------------------------
// Standalone operator handle: only the operator part of DevPlan is populated.
// ---------------------------------------------------------------------------
struct Operator {
  int device = 0;
  cudaStream_t stream = nullptr;
  DevPlan d{};
  void *arena = nullptr;
  double *pinned = nullptr;
  long long launches = 0;
};

static int op_create(int64_t n, const int64_t *rp, const int64_t *ci, int sym, int device,
                     Operator *&out) {
  out = nullptr;
  if (n < 0 || n >= INT32_MAX / 2) return set_error(KKT_ERR_BAD_SHAPE, "bad operator dimension");
  const int64_t nnz = rp[n];
  // general pattern + source map (the value-moving half of to_general, sparsecore.py:263)
  std::vector<int64_t> grp(n + 1, 0), gci, src;
  if (sym) {
    for (int64_t i = 0; i < n; ++i)
      for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
        if (ci[p] > i) return set_error(KKT_ERR_BAD_SHAPE, "entry above diagonal in symmetric-lower storage");
        grp[i + 1]++;
        if (ci[p] != i) grp[ci[p] + 1]++;
      }
    for (int64_t i = 0; i < n; ++i) grp[i + 1] += grp[i];
    gci.resize(grp[n]);
    src.resize(grp[n]);
    std::vector<int64_t> fill(grp.begin(), grp.end() - 1);
    // row-major sweep: row i gets its lower entries (cols ascending <= i) ...
    // ... and mirrored entries (i, k) for k > i arrive in ascending k => sorted rows.
    for (int64_t i = 0; i < n; ++i)
      for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
        int64_t q = fill[i]++;
        gci[q] = ci[p];
        src[q] = p;
      }
    for (int64_t i = 0; i < n; ++i)
      for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
        if (ci[p] != i) {
          int64_t q = fill[ci[p]]++;
          gci[q] = i;
          src[q] = p;
        }
    // rows now hold [lower part ascending][mirrored part ascending] = ascending overall
  } else {
    grp.assign(rp, rp + n + 1);
    gci.assign(ci, ci + nnz);
    src.resize(nnz);
    for (int64_t e = 0; e < nnz; ++e) src[e] = e;
  }
  const int64_t ng = grp[n];
  if (ng >= INT32_MAX) return set_error(KKT_ERR_BAD_SHAPE, "operator too large");
  std::vector<int> split(n);
  for (int64_t i = 0; i < n; ++i) {
    int64_t p = grp[i];
    while (p < grp[i + 1] && gci[p] <= i) ++p;
    split[i] = (int)p;
  }
  Operator *op = new Operator();
  op->device = device;
  cudaError_t ce = cudaSetDevice(device);
  if (ce == cudaSuccess) ce = cudaStreamCreateWithFlags(&op->stream, cudaStreamNonBlocking);
  if (ce != cudaSuccess) {
    delete op;
    return set_error(KKT_ERR_CUDA, std::string("operator stream: ") + cudaGetErrorString(ce));
  }
  DevPlan &d = op->d;
  d.n = (int)n;
  d.nnz_a = ng;
  d.in_nnz = nnz;
  d.sym_lower = sym ? 1 : 0;
  d.has_lower = sym ? 1 : 0;
  size_t bytes = 0;
  auto acc = [&](size_t b) { bytes += align_up(b + 1); };
  acc(4 * (n + 1)); acc(4 * ng); acc(4 * n); acc(4 * ng); acc(8 * std::max(nnz, ng)); acc(8 * ng);
  acc(8 * 32); acc(8 * 8 * RED_BLOCKS);
  ce = cudaMalloc(&op->arena, bytes);
  if (ce != cudaSuccess) {
    cudaStreamDestroy(op->stream);
    delete op;
    return set_error(KKT_ERR_OOM, "cudaMalloc of the operator failed");
  }
  char *cur = (char *)op->arena;
  d.A_rp = carve<int>(cur, n + 1);
  d.A_ci = carve<int>(cur, ng);
  d.A_split = carve<int>(cur, n);
  d.gen_src = carve<int>(cur, ng);
  d.in_vals = carve<double>(cur, std::max(nnz, ng));
  d.A_vals = carve<double>(cur, ng);
  d.scal = carve<unsigned long long>(cur, 32);
  d.partials = carve<double>(cur, 8 * RED_BLOCKS);
  std::vector<int> a = narrow<int64_t, int>(grp), b = narrow<int64_t, int>(gci), c = narrow<int64_t, int>(src);
  cudaMemcpyAsync(d.A_rp, a.data(), 4 * a.size(), cudaMemcpyHostToDevice, op->stream);
  cudaMemcpyAsync(d.A_ci, b.data(), 4 * b.size(), cudaMemcpyHostToDevice, op->stream);
  cudaMemcpyAsync(d.A_split, split.data(), 4 * split.size(), cudaMemcpyHostToDevice, op->stream);
  cudaMemcpyAsync(d.gen_src, c.data(), 4 * c.size(), cudaMemcpyHostToDevice, op->stream);
  cudaMemsetAsync(d.scal, 0, 8 * 32, op->stream);
  ce = cudaMallocHost(&op->pinned, 4096);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(op->stream);
  if (ce != cudaSuccess) {
    cudaFree(op->arena);
    cudaStreamDestroy(op->stream);
    delete op;
    return set_error(KKT_ERR_CUDA, std::string("operator upload: ") + cudaGetErrorString(ce));
  }
  out = op;
  return KKT_OK;
}

}  // namespace kkt

// ============================================================================
// C ABI
// ============================================================================
using kkt::Device;

extern "C" {

int kkt_dev_create(const kkt_symbolic *s, const int64_t *A_row_ptr, const int64_t *A_col_idx,
                   int64_t in_nnz, const int64_t *gen_src, const kkt_device_opts *opts,
                   kkt_device **out) {
  if (!s || !out || !A_row_ptr || !A_col_idx) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  *out = nullptr;
  try {
    Device *dev = nullptr;
    int rc = kkt::create(*reinterpret_cast<const kkt::Symbolic *>(s), A_row_ptr, A_col_idx, in_nnz,
                         gen_src, opts, dev);
    if (rc != KKT_OK) return rc;
    *out = reinterpret_cast<kkt_device *>(dev);
    return KKT_OK;
  } catch (std::bad_alloc &) {
    return kkt::set_error(KKT_ERR_OOM, "host allocation failed in kkt_dev_create");
  }
}

void kkt_dev_destroy(kkt_device *d) { kkt::destroy(reinterpret_cast<Device *>(d)); }

void *kkt_dev_stream(kkt_device *d) { return d ? (void *)reinterpret_cast<Device *>(d)->stream : nullptr; }

int kkt_dev_refactor(kkt_device *d, const double *values_in, int layout, int values_on_device,
                     double *diag_out) {
  Device *dev = reinterpret_cast<Device *>(d);
  if (!dev || !values_in) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(dev->device);
  return kkt::refactor(dev, values_in, layout, values_on_device, diag_out);
}

int kkt_dev_set_operator_values(kkt_device *d, const double *values_in, int layout,
                                int values_on_device) {
  Device *dev = reinterpret_cast<Device *>(d);
  if (!dev || !values_in) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(dev->device);
  return kkt::set_values(dev, values_in, layout, values_on_device);
}

int kkt_dev_download_factors(kkt_device *d, double *Lx, double *Ux, double *Udiag) {
  Device *dev = reinterpret_cast<Device *>(d);
  if (!dev) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(dev->device);
  const kkt::DevPlan &p = dev->d;
  cudaStream_t s = dev->stream;
  cudaError_t e = cudaSuccess;
  if (Lx && p.nnz_L) e = cudaMemcpyAsync(Lx, p.Lx, 8 * (size_t)p.nnz_L, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && Ux && p.nnz_U) e = cudaMemcpyAsync(Ux, p.Ux, 8 * (size_t)p.nnz_U, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && Udiag && p.n) e = cudaMemcpyAsync(Udiag, p.udiag, 8 * (size_t)p.n, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return kkt::set_error(KKT_ERR_CUDA, cudaGetErrorString(e));
  return KKT_OK;
}

int kkt_dev_solve(kkt_device *d, const double *b_dev, double *x_dev) {
  Device *dev = reinterpret_cast<Device *>(d);
  if (!dev || !b_dev || !x_dev) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(dev->device);
  return kkt::solve(dev, b_dev, x_dev);
}

int kkt_dev_spmv(kkt_device *d, const double *x_dev, double *y_dev) {
  Device *dev = reinterpret_cast<Device *>(d);
  if (!dev || !x_dev || !y_dev) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(dev->device);
  return kkt::spmv(dev, x_dev, y_dev, nullptr, nullptr);
}

int kkt_dev_residual_norms(kkt_device *d, const double *r_dev, const double *x_dev, double *out_host) {
  Device *dev = reinterpret_cast<Device *>(d);
  if (!dev || !r_dev || !x_dev || !out_host) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(dev->device);
  return kkt::residual_norms(dev, r_dev, x_dev, out_host);
}

int kkt_dev_fgmres(kkt_device *d, const double *b_dev, const double *x0_dev, double *x_dev,
                   const kkt_krylov_cfg *cfg, kkt_krylov_report *rep, double *history_host, int hist_cap) {
  Device *dev = reinterpret_cast<Device *>(d);
  if (!dev || !b_dev || !x0_dev || !x_dev || !cfg || !rep)
    return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(dev->device);
  return kkt::fgmres(dev, b_dev, x0_dev, x_dev, cfg, rep, history_host, hist_cap);
}

int kkt_dev_refine_fgmres(kkt_device *d, const double *r_dev, const double *x0_dev, double *x_dev,
                          const kkt_krylov_cfg *cfg, kkt_krylov_report *rep) {
  Device *dev = reinterpret_cast<Device *>(d);
  if (!dev || !r_dev || !x0_dev || !x_dev || !cfg || !rep)
    return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  if (!(cfg->delta_tol > 0)) return kkt::set_error(KKT_ERR_BAD_ARG, "delta_tol must be positive");
  cudaSetDevice(dev->device);
  double st[6];
  int rc = kkt::residual_norms(dev, r_dev, x0_dev, st);
  if (rc) return rc;
  std::memset(rep, 0, sizeof *rep);
  // needs_refinement: ||r - K x0||_2 > delta * ||r||_2   (refine.py:88-92)
  if (!(st[0] > cfg->delta_tol * st[4])) {
    cudaError_t e = cudaMemcpyAsync(x_dev, x0_dev, 8 * (size_t)dev->d.n, cudaMemcpyDeviceToDevice, dev->stream);
    if (e != cudaSuccess) return kkt::set_error(KKT_ERR_CUDA, cudaGetErrorString(e));
    rep->triggered = 0;
    rep->converged = 1;
    return KKT_OK;
  }
  kkt_krylov_cfg c = *cfg;
  c.tol = cfg->delta_tol;
  rc = kkt::fgmres(dev, r_dev, x0_dev, x_dev, &c, rep, nullptr, 0);
  rep->triggered = 1;
  return rc;
}

int kkt_dev_step(kkt_device *d, const double *values_in, int layout, const double *r_in,
                 double *x_out, int io_on_device, const kkt_krylov_cfg *cfg, kkt_krylov_report *rep,
                 double *diag_out) {
  Device *dev = reinterpret_cast<Device *>(d);
  if (!dev || !values_in || !r_in || !x_out || !cfg || !rep)
    return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(dev->device);
  int rc = kkt::refactor(dev, values_in, layout, io_on_device, diag_out);
  if (rc) return rc;
  kkt::Krylov &K = *dev->kry;
  const size_t nb = 8 * (size_t)dev->d.n;
  const double *r_dev = r_in;
  if (!io_on_device) {
    cudaError_t e = cudaMemcpyAsync(K.sr, r_in, nb, cudaMemcpyHostToDevice, dev->stream);
    if (e != cudaSuccess) return kkt::set_error(KKT_ERR_CUDA, cudaGetErrorString(e));
    r_dev = K.sr;
  }
  rc = kkt::solve(dev, r_dev, K.sx0);  // x0 = lu_solve(r)      (harness.py:234)
  if (rc) return rc;
  rc = kkt_dev_refine_fgmres(d, r_dev, K.sx0, K.sx, cfg, rep);  // (harness.py:240)
  if (rc) return rc;
  cudaError_t e = cudaMemcpyAsync(x_out, K.sx, nb,
                                  io_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                  dev->stream);
  if (e != cudaSuccess) return kkt::set_error(KKT_ERR_CUDA, cudaGetErrorString(e));
  e = cudaStreamSynchronize(dev->stream);
  if (e != cudaSuccess) return kkt::set_error(KKT_ERR_CUDA, cudaGetErrorString(e));
  return KKT_OK;
}

int kkt_op_create(int64_t n, const int64_t *row_ptr, const int64_t *col_idx, int symmetric_lower,
                  int device, kkt_operator **out) {
  if (!row_ptr || !out || (n > 0 && !col_idx)) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  *out = nullptr;
  try {
    kkt::Operator *op = nullptr;
    int rc = kkt::op_create(n, row_ptr, col_idx, symmetric_lower, device, op);
    if (rc) return rc;
    *out = reinterpret_cast<kkt_operator *>(op);
    return KKT_OK;
  } catch (std::bad_alloc &) {
    return kkt::set_error(KKT_ERR_OOM, "host allocation failed in kkt_op_create");
  }
}

void kkt_op_destroy(kkt_operator *o) {
  kkt::Operator *op = reinterpret_cast<kkt::Operator *>(o);
  if (!op) return;
  cudaSetDevice(op->device);
  cudaStreamSynchronize(op->stream);
  cudaFree(op->arena);
  cudaFreeHost(op->pinned);
  cudaStreamDestroy(op->stream);
  delete op;
}

void *kkt_op_stream(kkt_operator *o) {
  return o ? (void *)reinterpret_cast<kkt::Operator *>(o)->stream : nullptr;
}

// The operator shares the kernels of the device handle through a lightweight Device view.
static kkt::Device op_view(kkt::Operator *op) {
  kkt::Device v;
  v.device = op->device;
  v.stream = op->stream;
  v.d = op->d;
  v.pinned = op->pinned;
  return v;
}

int kkt_op_set_values(kkt_operator *o, const double *values, int on_device) {
  kkt::Operator *op = reinterpret_cast<kkt::Operator *>(o);
  if (!op || !values) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(op->device);
  kkt::Device v = op_view(op);
  int rc = kkt::set_values(&v, values, op->d.has_lower ? KKT_LAYOUT_SYMMETRIC_LOWER : KKT_LAYOUT_GENERAL,
                           on_device);
  op->launches += v.launches;
  v.stream = nullptr;
  v.pinned = nullptr;
  return rc;
}

int kkt_op_spmv(kkt_operator *o, const double *x_dev, double *y_dev) {
  kkt::Operator *op = reinterpret_cast<kkt::Operator *>(o);
  if (!op || !x_dev || !y_dev) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(op->device);
  kkt::Device v = op_view(op);
  int rc = kkt::spmv(&v, x_dev, y_dev, nullptr, nullptr);
  op->launches += v.launches;
  v.stream = nullptr;
  v.pinned = nullptr;
  return rc;
}

int kkt_op_residual_norms(kkt_operator *o, const double *r_dev, const double *x_dev, double *out_host) {
  kkt::Operator *op = reinterpret_cast<kkt::Operator *>(o);
  if (!op || !r_dev || !x_dev || !out_host) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(op->device);
  kkt::Device v = op_view(op);
  int rc = kkt::residual_norms(&v, r_dev, x_dev, out_host);
  op->launches += v.launches;
  v.stream = nullptr;
  v.pinned = nullptr;
  return rc;
}

int64_t kkt_dev_launch_count(kkt_device *d) {
  return d ? reinterpret_cast<Device *>(d)->launches : 0;
}

}  // extern "C"
