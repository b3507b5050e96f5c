// Restarted right-preconditioned FGMRES(m) with CGS2 (krylov.fgmres / cgs2_step,
// krylov.py:93-208) on the device.  Per iteration: z = M v (triangular solves),
// w = K z (SpMV), CGS2 as two (multi-dot, fused multi-axpy) passes — the second pass also
// produces ||w||^2 — then the Hessenberg/Givens update in a one-thread kernel that publishes
// the residual estimate and the stop flag.  The host reads one 32-byte status per iteration
// (the reference's per-iteration convergence test); no vector ever leaves HBM.
#include <cuda_runtime.h>

#include <cstring>

#include "host_util.h"
#include "kernels.cuh"

namespace kkt {

// h[q] = V_q . w for q < nvec as block partials (vectors in groups of 8, w re-read from L2).
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

// w_out = w_in - sum_q V_q h[q]; mode 1 also emits ||w_out||^2 block partials.
__global__ void __launch_bounds__(RED_THREADS) k_cgs(const double *__restrict__ V, int nvec, int n,
                                                     const double *__restrict__ w_in,
                                                     const double *__restrict__ h,
                                                     double *__restrict__ w_out, int mode,
                                                     double *__restrict__ partials) {
  __shared__ double sh[32];
  __shared__ double hs[64];
  for (int q = threadIdx.x; q < nvec; q += blockDim.x) hs[q] = h[q];
  __syncthreads();
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double t = 0.0;
    for (int q = 0; q < nvec; ++q) t += V[(size_t)q * n + i] * hs[q];
    const double o = w_in[i] - t;
    w_out[i] = o;
    acc += o * o;
  }
  if (mode == 1) {
    const double t = block_sum<RED_THREADS>(acc, sh);
    if (threadIdx.x == 0) partials[blockIdx.x] = t;
  }
}

// Hessenberg column j, previous rotations, new rotation, residual estimate (:166-186).
__global__ void k_givens(KState *st, int j, int m, const double *__restrict__ h1,
                         const double *__restrict__ h2, const double *__restrict__ nrm2,
                         double *H, double *cs, double *sn, double *g, double *status) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int i = 0; i <= j; ++i) H[i * m + j] = h1[i] + h2[i];  // H is (m+1) x m row-major
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

void free_krylov(Device *dev) {
  if (dev->kry) {
    cudaFree(dev->kry->mem);
    delete dev->kry;
    dev->kry = nullptr;
  }
}

int alloc_krylov(Device *dev, int m) {
  Krylov *K = new Krylov();
  K->m = m;
  K->n = dev->d.n;
  const size_t n = (size_t)dev->d.n;
  size_t bytes = align_up(8 * (m + 1) * n + 1) + align_up(8 * m * n + 1) + 7 * align_up(8 * n + 1);
  bytes += 6 * align_up(8 * (m + 1) + 1) + align_up(8 * (m + 1) * m + 1) + 2 * align_up(64 + 1);
  bytes += align_up(sizeof(KState) + 1) + align_up(8 * (m + 2) * RED_BLOCKS + 1);
  if (cudaMalloc(&K->mem, bytes) != cudaSuccess) {
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
  K->cs = carve<double>(cur, m + 1);
  K->sn = carve<double>(cur, m + 1);
  K->g = carve<double>(cur, m + 1);
  K->yv = carve<double>(cur, m + 1);
  K->H = carve<double>(cur, (size_t)(m + 1) * m);
  K->nrm = carve<double>(cur, 8);
  K->beta = carve<double>(cur, 8);
  K->st = carve<KState>(cur, 1);
  K->partials = carve<double>(cur, (size_t)(m + 2) * RED_BLOCKS);
  free_krylov(dev);
  dev->kry = K;
  return KKT_OK;
}

// Read `count` doubles (device) + the non-finite flag into pinned memory; one sync.
static int read_status(Device *dev, const double *src, int count, bool *nonfinite) {
  if (count) CUDA_TRY(cudaMemcpyAsync(dev->pinned, src, 8 * count, cudaMemcpyDeviceToHost, dev->stream));
  CUDA_TRY(cudaMemcpyAsync(dev->pinned + 8, &dev->d.scal[SC_NONFINITE], 8, cudaMemcpyDeviceToHost,
                           dev->stream));
  CUDA_TRY(cudaStreamSynchronize(dev->stream));
  unsigned long long f;
  std::memcpy(&f, dev->pinned + 8, 8);
  *nonfinite = f != 0;
  return KKT_OK;
}

int dev_fgmres(Device *dev, const double *b, const double *x0, double *xout,
               const kkt_krylov_cfg *cfg, kkt_krylov_report *rep, double *hist, int hist_cap) {
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
  cudaStream_t s = dev->stream;
  std::memset(rep, 0, sizeof *rep);
  int hn = 0;
  auto push_hist = [&](double v) {
    if (hist && hn < hist_cap) hist[hn] = v;
    hn++;
  };
  bool nonfinite = false;
  CUDA_TRY(cudaMemsetAsync(&d.scal[SC_NONFINITE], 0, 8, s));
  CUDA_TRY(cudaMemcpyAsync(K.x, x0, 8 * (size_t)n, cudaMemcpyDeviceToDevice, s));
  // r = b - K x; beta0 = ||r||                                           (:133-134)
  int rc = dev_spmv(dev, K.x, K.r, b, K.partials);
  if (rc) return rc;
  LAUNCH(launch_reduce_partials(K.partials, 1, RED_BLOCKS, K.beta, 1, s));
  if ((rc = read_status(dev, K.beta, 1, &nonfinite))) return rc;
  if (nonfinite) {
    rep->nonfinite = 1;
    return set_error(KKT_ERR_NONFINITE, "operator produced a non-finite entry");
  }
  const double beta0 = dev->pinned[0];
  push_hist(beta0);
  rep->beta0 = beta0;
  if (beta0 == 0.0) {  // (:140-141)
    CUDA_TRY(cudaMemcpyAsync(xout, K.x, 8 * (size_t)n, cudaMemcpyDeviceToDevice, s));
    rep->converged = 1;
    rep->est_final = beta0;
    return KKT_OK;
  }
  KState st{};
  st.beta0 = beta0;
  st.target = cfg->tol * beta0;
  st.floor = HAPPY_BREAKDOWN_RTOL * beta0;
  CUDA_TRY(cudaMemcpyAsync(K.st, &st, sizeof st, cudaMemcpyHostToDevice, s));
  double beta = beta0, est = beta0;
  int converged = 0, iters = 0, restarts = 0;
  const int G = RED_BLOCKS, T = RED_THREADS;
  double *status = K.partials + (size_t)(m + 1) * RED_BLOCKS;
  for (int outer = 0; outer < cfg->max_outer; ++outer) {
    if (beta <= st.target) {  // (:148-150)
      converged = 1;
      break;
    }
    k_scale<<<G, T, 0, s>>>(K.r, K.V, n, K.beta);  // V0 = r / beta (a division, :151)
    LAUNCH(cudaGetLastError());
    k_cycle_init<<<1, 128, 0, s>>>(K.g, m, K.beta, K.H);
    LAUNCH(cudaGetLastError());
    int j_used = 0;
    bool stop = false;
    for (int j = 0; j < m; ++j) {
      double *Vj = K.V + (size_t)j * n;
      double *Zj = K.Z + (size_t)j * n;
      if ((rc = dev_solve(dev, Vj, Zj))) return rc;                    // z = M(V_j)   :161
      if ((rc = dev_spmv(dev, Zj, K.w, nullptr, nullptr))) return rc;  // w = K z      :163
      const int nv = j + 1;
      // cgs2_step (:93-105): h1 = V^T w; w1 = w - V h1; h2 = V^T w1; w2 = w1 - V h2
      k_dots<<<G, T, 0, s>>>(K.V, nv, n, K.w, K.partials);
      LAUNCH(cudaGetLastError());
      LAUNCH(launch_reduce_partials(K.partials, nv, RED_BLOCKS, K.h1, 0, s));
      k_cgs<<<G, T, 0, s>>>(K.V, nv, n, K.w, K.h1, K.w1, 0, nullptr);
      LAUNCH(cudaGetLastError());
      k_dots<<<G, T, 0, s>>>(K.V, nv, n, K.w1, K.partials);
      LAUNCH(cudaGetLastError());
      LAUNCH(launch_reduce_partials(K.partials, nv, RED_BLOCKS, K.h2, 0, s));
      k_cgs<<<G, T, 0, s>>>(K.V, nv, n, K.w1, K.h2, K.w, 1, K.partials);
      LAUNCH(cudaGetLastError());
      LAUNCH(launch_reduce_partials(K.partials, 1, RED_BLOCKS, K.nrm, 0, s));
      k_givens<<<1, 32, 0, s>>>(K.st, j, m, K.h1, K.h2, K.nrm, K.H, K.cs, K.sn, K.g, status);
      LAUNCH(cudaGetLastError());
      if ((rc = read_status(dev, status, 3, &nonfinite))) return rc;
      if (nonfinite) {
        rep->nonfinite = 1;
        rep->iterations = iters;
        return set_error(KKT_ERR_NONFINITE, "preconditioner or operator produced a non-finite entry");
      }
      est = dev->pinned[0];
      stop = dev->pinned[1] != 0.0;
      push_hist(est);
      iters++;
      j_used = j + 1;
      if (stop) break;  // est <= target or happy breakdown (:184-186)
      k_scale<<<G, T, 0, s>>>(K.w, K.V + (size_t)(j + 1) * n, n, status + 2);  // V_{j+1} = w/hj1
      LAUNCH(cudaGetLastError());
    }
    // y = R^{-1} g; x += Z y; r = b - K x; beta = ||r||                    (:189-192)
    k_solve_upper<<<1, 32, 0, s>>>(K.H, m, K.g, j_used, K.yv);
    LAUNCH(cudaGetLastError());
    k_update_x<<<G, T, 0, s>>>(K.x, K.Z, n, K.yv, j_used);
    LAUNCH(cudaGetLastError());
    if ((rc = dev_spmv(dev, K.x, K.r, b, K.partials))) return rc;
    LAUNCH(launch_reduce_partials(K.partials, 1, RED_BLOCKS, K.beta, 1, s));
    if ((rc = read_status(dev, K.beta, 1, &nonfinite))) return rc;
    if (nonfinite) {
      rep->nonfinite = 1;
      return set_error(KKT_ERR_NONFINITE, "operator produced a non-finite entry");
    }
    beta = dev->pinned[0];
    restarts++;
    if (stop || beta <= st.target) {  // (:194-198)
      converged = 1;
      break;
    }
  }
  CUDA_TRY(cudaMemcpyAsync(xout, K.x, 8 * (size_t)n, cudaMemcpyDeviceToDevice, s));
  rep->iterations = iters;
  rep->precond_applications = iters;
  rep->converged = converged;
  rep->restarts = restarts;
  rep->est_final = est;
  rep->true_final = beta;
  return KKT_OK;
}

}  // namespace kkt
