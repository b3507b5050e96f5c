// Restarted right-preconditioned FGMRES(m) with CGS2 (krylov.fgmres / cgs2_step,
// krylov.py:93-208) on the device, for nb same-pattern systems at once.
//
// Per iteration: z = M v (triangular solves, all systems in one launch), w = K z (SpMV),
// CGS2 as two (multi-dot, fused multi-axpy) passes — the second also produces ||w||^2 —
// then the Hessenberg/Givens update in a one-warp-per-system kernel that publishes the
// residual estimate and the stop flag.  Systems advance in lockstep cycles; each keeps the
// reference's own semantics (stop inside a cycle on est <= tol*beta0 or happy breakdown,
// solution + true residual at the cycle end, restart budget) through a per-system mask.
// The host reads one small status block per iteration; no vector ever leaves HBM.
// Layouts: V [m+1][nb][n], Z [m][nb][n] (the j-th basis of all systems is contiguous, which
// is the [nb][n] layout the solve and SpMV consume); per-system small state [nb][...].
#include <cuda_runtime.h>

#include <cstring>
#include <vector>

#include "host_util.h"
#include "kernels.cuh"

namespace kkt {

// h[q] = V_q . w (q < nvec) as block partials [nb][nvec][rb]; skipped for masked systems.
__global__ void __launch_bounds__(RED_THREADS) k_dots(const double *__restrict__ V, int nb, int nvec,
                                                      int n, const double *__restrict__ w,
                                                      const int *__restrict__ mask,
                                                      double *__restrict__ partials) {
  __shared__ double sh[32];
  const int sys = blockIdx.y;
  if (!mask[sys]) return;
  const double *ws = w + (size_t)sys * n;
  for (int g0 = 0; g0 < nvec; g0 += 8) {
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int gn = min(8, nvec - g0);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
      const double wi = ws[i];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < gn) acc[q] += V[((size_t)(g0 + q) * nb + sys) * n + i] * wi;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (q < gn) {
        const double t = block_sum<RED_THREADS>(acc[q], sh);
        if (threadIdx.x == 0) partials[((size_t)sys * nvec + g0 + q) * gridDim.x + blockIdx.x] = t;
      }
    }
  }
}

// w_out = w_in - sum_q V_q h[q]; mode 1 also emits ||w_out||^2 block partials [nb][rb].
__global__ void __launch_bounds__(RED_THREADS) k_cgs(const double *__restrict__ V, int nb, int nvec,
                                                     int n, const double *__restrict__ w_in,
                                                     const double *__restrict__ h, int hstride,
                                                     double *__restrict__ w_out, int mode,
                                                     const int *__restrict__ mask,
                                                     double *__restrict__ partials) {
  __shared__ double sh[32];
  __shared__ double hs[64];
  const int sys = blockIdx.y;
  if (!mask[sys]) return;
  for (int q = threadIdx.x; q < nvec; q += blockDim.x) hs[q] = h[(size_t)sys * hstride + q];
  __syncthreads();
  const double *wi_ = w_in + (size_t)sys * n;
  double *wo_ = w_out + (size_t)sys * n;
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double t = 0.0;
    for (int q = 0; q < nvec; ++q) t += V[((size_t)q * nb + sys) * n + i] * hs[q];
    const double o = wi_[i] - t;
    wo_[i] = o;
    acc += o * o;
  }
  if (mode == 1) {
    const double t = block_sum<RED_THREADS>(acc, sh);
    if (threadIdx.x == 0) partials[(size_t)sys * gridDim.x + blockIdx.x] = t;
  }
}

// Per system: Hessenberg column j, previous rotations, new rotation, estimate (:166-186).
// status[sys] = {est, stop, hj1, nonfinite}.
__global__ void k_givens(KState *st, int j, int m, const double *__restrict__ h1,
                         const double *__restrict__ h2, const double *__restrict__ nrm2,
                         double *H, double *cs, double *sn, double *g, double *status,
                         const int *__restrict__ mask, const unsigned long long *scal) {
  const int sys = blockIdx.x;
  if (threadIdx.x != 0) return;
  double *stat = status + 4 * sys;
  stat[3] = scal[(size_t)sys * SCAL_STRIDE + SC_NONFINITE] ? 1.0 : 0.0;
  if (!mask[sys]) return;
  const int m1 = m + 1;
  double *Hs = H + (size_t)sys * m1 * m;
  double *css = cs + (size_t)sys * m1, *sns = sn + (size_t)sys * m1, *gs = g + (size_t)sys * m1;
  KState *S = st + sys;
  for (int i = 0; i <= j; ++i) Hs[i * m + j] = h1[(size_t)sys * m1 + i] + h2[(size_t)sys * m1 + i];
  const double hj1 = sqrt(nrm2[sys]);
  Hs[(j + 1) * m + j] = hj1;
  for (int i = 0; i < j; ++i) {
    const double a = Hs[i * m + j], b = Hs[(i + 1) * m + j];
    const double t = __dadd_rn(__dmul_rn(css[i], a), __dmul_rn(sns[i], b));
    Hs[(i + 1) * m + j] = __dadd_rn(__dmul_rn(-sns[i], a), __dmul_rn(css[i], b));
    Hs[i * m + j] = t;
  }
  const double denom = hypot(Hs[j * m + j], Hs[(j + 1) * m + j]);
  css[j] = __ddiv_rn(Hs[j * m + j], denom);
  sns[j] = __ddiv_rn(Hs[(j + 1) * m + j], denom);
  Hs[j * m + j] = denom;
  Hs[(j + 1) * m + j] = 0.0;
  gs[j + 1] = __dmul_rn(-sns[j], gs[j]);
  gs[j] = __dmul_rn(css[j], gs[j]);
  const double est = fabs(gs[j + 1]);
  S->est = est;
  S->hj1 = hj1;
  S->j = j;
  const int stop = (est <= S->target || hj1 <= S->floor) ? 1 : 0;
  S->stop = stop;
  stat[0] = est;
  stat[1] = stop;
  stat[2] = hj1;
}

// status[sys] = {beta[sys] (if given), -, -, nonfinite flag}
__global__ void k_status(double *status, const unsigned long long *scal, const double *beta, int nb) {
  for (int q = threadIdx.x; q < nb; q += blockDim.x) {
    if (beta) status[4 * q] = beta[q];
    status[4 * q + 3] = scal[(size_t)q * SCAL_STRIDE + SC_NONFINITE] ? 1.0 : 0.0;
  }
}

// out_sys = in_sys / den[sys * dstride] for systems in the mask
__global__ void k_scale(const double *__restrict__ in, double *__restrict__ out, int n,
                        const double *__restrict__ den, int dstride, const int *__restrict__ mask) {
  const int sys = blockIdx.y;
  if (!mask[sys]) return;
  const double dv = den[(size_t)sys * dstride];
  const double *is = in + (size_t)sys * n;
  double *os = out + (size_t)sys * n;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    os[i] = __ddiv_rn(is[i], dv);
}

__global__ void k_cycle_init(double *g, double *H, int m, const double *beta, const int *mask,
                             unsigned long long *scal) {
  const int sys = blockIdx.x;
  if (!mask[sys]) return;
  double *gs = g + (size_t)sys * (m + 1);
  double *Hs = H + (size_t)sys * (m + 1) * m;
  for (int i = threadIdx.x; i <= m; i += blockDim.x) gs[i] = (i == 0) ? beta[sys] : 0.0;
  for (int i = threadIdx.x; i < (m + 1) * m; i += blockDim.x) Hs[i] = 0.0;
  if (threadIdx.x == 0) scal[(size_t)sys * SCAL_STRIDE + SC_NONFINITE] = 0ull;
}

// y = R^{-1} g on the leading k x k block, k = jused[sys] (krylov.py:211-216).
__global__ void k_solve_upper(const double *H, int m, const double *g, const int *jused, double *y) {
  const int sys = blockIdx.x;
  if (threadIdx.x != 0) return;
  const int k = jused[sys];
  const double *Hs = H + (size_t)sys * (m + 1) * m;
  const double *gs = g + (size_t)sys * (m + 1);
  double *ys = y + (size_t)sys * (m + 1);
  for (int i = k - 1; i >= 0; --i) {
    double dot = 0.0;
    for (int q = i + 1; q < k; ++q) dot = __dadd_rn(dot, __dmul_rn(Hs[i * m + q], ys[q]));
    ys[i] = __ddiv_rn(__dsub_rn(gs[i], dot), Hs[i * m + i]);
  }
}

// x = x + (sum_q Z_q y_q) for k = jused[sys] (krylov.py:190: the matvec first, then the add)
__global__ void k_update_x(double *__restrict__ x, const double *__restrict__ Z, int nb, int n,
                           const double *__restrict__ y, int ystride, const int *__restrict__ jused) {
  const int sys = blockIdx.y;
  const int k = jused[sys];
  if (!k) return;
  double *xs = x + (size_t)sys * n;
  const double *ys = y + (size_t)sys * ystride;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double t = 0.0;
    for (int q = 0; q < k; ++q) t = __dadd_rn(t, __dmul_rn(Z[((size_t)q * nb + sys) * n + i], ys[q]));
    xs[i] = __dadd_rn(xs[i], t);
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
  const size_t n = (size_t)dev->d.n, nb = (size_t)dev->d.nbp, rb = (size_t)dev->d.rb;
  size_t bytes = align_up(8 * (m + 1) * nb * n + 1) + align_up(8 * m * nb * n + 1) +
                 7 * align_up(8 * nb * n + 1);
  bytes += 6 * align_up(8 * nb * (m + 1) + 1) + align_up(8 * nb * (m + 1) * m + 1);
  bytes += 2 * align_up(8 * nb + 64) + align_up(sizeof(KState) * nb + 1);
  bytes += align_up(8 * (m + 2) * rb * nb + 1) + align_up(8 * 4 * nb + 1) + 2 * align_up(4 * nb + 1);
  if (cudaMalloc(&K->mem, bytes) != cudaSuccess) {
    delete K;
    return set_error(KKT_ERR_OOM, "cudaMalloc of the FGMRES workspace failed");
  }
  cudaMemsetAsync(K->mem, 0, bytes, dev->stream);
  char *cur = (char *)K->mem;
  K->V = carve<double>(cur, (m + 1) * nb * n);
  K->Z = carve<double>(cur, (size_t)m * nb * n);
  K->w = carve<double>(cur, nb * n);
  K->w1 = carve<double>(cur, nb * n);
  K->r = carve<double>(cur, nb * n);
  K->x = carve<double>(cur, nb * n);
  K->sr = carve<double>(cur, nb * n);
  K->sx0 = carve<double>(cur, nb * n);
  K->sx = carve<double>(cur, nb * n);
  K->h1 = carve<double>(cur, nb * (m + 1));
  K->h2 = carve<double>(cur, nb * (m + 1));
  K->cs = carve<double>(cur, nb * (m + 1));
  K->sn = carve<double>(cur, nb * (m + 1));
  K->g = carve<double>(cur, nb * (m + 1));
  K->yv = carve<double>(cur, nb * (m + 1));
  K->H = carve<double>(cur, nb * (m + 1) * m);
  K->nrm = carve<double>(cur, nb + 8);
  K->beta = carve<double>(cur, nb + 8);
  K->st = carve<KState>(cur, nb);
  K->partials = carve<double>(cur, (m + 2) * rb * nb);
  K->status = carve<double>(cur, 4 * nb);
  K->mask = carve<int>(cur, nb);
  K->jused = carve<int>(cur, nb);
  free_krylov(dev);
  dev->kry = K;
  return KKT_OK;
}

// Copy `count` doubles from the device into pinned memory; one stream sync.
static int read_block(Device *dev, const double *src, size_t count) {
  if (8 * count > dev->pinned_bytes) return set_error(KKT_ERR_BAD_ARG, "status block too large");
  CUDA_TRY(cudaMemcpyAsync(dev->pinned, src, 8 * count, cudaMemcpyDeviceToHost, dev->stream));
  CUDA_TRY(cudaStreamSynchronize(dev->stream));
  return KKT_OK;
}

// per-system int flags [nb] -> device [nbp] (padding systems are never active).  A pageable
// source: cudaMemcpyAsync has consumed it when it returns.
static int upload_mask(Device *dev, const std::vector<int> &mask, int *dst) {
  std::vector<int> pad(dev->d.nbp, 0);
  for (size_t q = 0; q < mask.size() && q < pad.size(); ++q) pad[q] = mask[q];
  CUDA_TRY(cudaMemcpyAsync(dst, pad.data(), 4 * pad.size(), cudaMemcpyHostToDevice, dev->stream));
  return KKT_OK;
}

int dev_fgmres(Device *dev, const double *b, const double *x0, double *xout,
               const kkt_krylov_cfg *cfg, kkt_krylov_report *rep, double *hist, int hist_cap,
               const int *active_in) {
  DevPlan &d = dev->d;
  const int n = d.n, nb = d.nb;
  if (cfg->m < 1) return set_error(KKT_ERR_BAD_ARG, "restart length m must be >= 1");
  if (!(cfg->tol > 0)) return set_error(KKT_ERR_BAD_ARG, "tol must be positive");
  if (cfg->m > 62) return set_error(KKT_ERR_BAD_ARG, "restart length m must be <= 62");
  if (!dev->kry || dev->kry->m < cfg->m) {
    int rc = alloc_krylov(dev, cfg->m);
    if (rc != KKT_OK) return rc;
  }
  Krylov &K = *dev->kry;
  const int m = cfg->m, M = K.m;  // M: workspace stride (>= m)
  struct MaskGuard {  // the solves/SpMVs below only touch the running systems
    DevPlan &d;
    ~MaskGuard() { d.sys_mask = nullptr; }
  } guard{d};
  cudaStream_t s = dev->stream;
  const size_t nbn = (size_t)d.nbp * n;
  const bool il = d.nbp > 1;
  std::vector<int> hn(nb, 0), active(nb, 1), running(nb, 0), jused(nb, 0);
  std::vector<double> beta(nb, 0.0), target(nb, 0.0), est(nb, 0.0);
  std::vector<int> iters(nb, 0), converged(nb, 0), restarts(nb, 0);
  for (int q = 0; q < nb; ++q) {
    std::memset(&rep[q], 0, sizeof rep[q]);
    if (active_in) active[q] = active_in[q] ? 1 : 0;
  }
  auto push_hist = [&](int q, double v) {
    if (hist && hn[q] < hist_cap) hist[(size_t)q * hist_cap + hn[q]] = v;
    hn[q]++;
  };
  auto fail_nonfinite = [&](int q) {
    rep[q].nonfinite = 1;
    return set_error(KKT_ERR_NONFINITE, "operator or preconditioner produced a non-finite entry");
  };
  for (int q = 0; q < nb; ++q) CUDA_TRY(cudaMemsetAsync(&d.scal[(size_t)q * SCAL_STRIDE + SC_NONFINITE], 0, 8, s));
  CUDA_TRY(cudaMemcpyAsync(K.x, x0, 8 * nbn, cudaMemcpyDeviceToDevice, s));
  // r = b - K x; beta0 = ||r||                                             (:133-134)
  int rc = dev_spmv(dev, K.x, K.r, b, K.partials);
  if (rc) return rc;
  LAUNCH(launch_reduce_partials(d, K.partials, 1, K.beta, 1, 1, s));
  LAUNCH((k_status<<<1, 64, 0, s>>>(K.status, d.scal, K.beta, nb), cudaGetLastError()));
  if ((rc = read_block(dev, K.status, 4 * nb))) return rc;
  for (int q = 0; q < nb; ++q) {
    beta[q] = dev->pinned[4 * q];
    if (active[q] && dev->pinned[4 * q + 3] != 0.0) return fail_nonfinite(q);
  }
  std::vector<KState> st(nb);
  for (int q = 0; q < nb; ++q) {
    rep[q].beta0 = beta[q];
    est[q] = beta[q];
    if (!active[q]) continue;
    push_hist(q, beta[q]);
    if (beta[q] == 0.0) {  // (:140-141)
      converged[q] = 1;
      active[q] = 0;
    }
    st[q] = KState{};
    st[q].beta0 = beta[q];
    const double tol_q = cfg->delta_sys ? cfg->delta_sys[q] : cfg->tol;
    st[q].target = target[q] = tol_q * beta[q];
    st[q].floor = HAPPY_BREAKDOWN_RTOL * beta[q];
  }
  CUDA_TRY(cudaMemcpyAsync(K.st, st.data(), sizeof(KState) * nb, cudaMemcpyHostToDevice, s));
  const int G = d.rb, T = RED_THREADS;
  for (int outer = 0; outer < cfg->max_outer; ++outer) {
    int any = 0;
    for (int q = 0; q < nb; ++q) {
      running[q] = 0;
      jused[q] = 0;
      if (!active[q]) continue;
      if (beta[q] <= target[q]) {  // (:148-150)
        converged[q] = 1;
        active[q] = 0;
        continue;
      }
      running[q] = 1;
      any = 1;
    }
    if (!any) break;
    if ((rc = upload_mask(dev, running, K.mask))) return rc;
    LAUNCH(il ? b_launch_scale(d, K.r, K.V, K.beta, 1, K.mask, s)
              : (k_scale<<<dim3(G, nb), T, 0, s>>>(K.r, K.V, n, K.beta, 1, K.mask), cudaGetLastError()));
    LAUNCH((k_cycle_init<<<nb, 128, 0, s>>>(K.g, K.H, M, K.beta, K.mask, d.scal), cudaGetLastError()));
    std::vector<int> cycle(running);
    for (int j = 0; j < m; ++j) {
      bool anyrun = false;
      for (int q = 0; q < nb; ++q) anyrun |= running[q] != 0;
      if (!anyrun) break;
      double *Vj = K.V + (size_t)j * nbn;
      double *Zj = K.Z + (size_t)j * nbn;
      d.sys_mask = K.mask;
      if ((rc = dev_solve(dev, Vj, Zj))) return rc;                    // z = M(V_j)   :161
      if ((rc = dev_spmv(dev, Zj, K.w, nullptr, nullptr))) return rc;  // w = K z      :163
      d.sys_mask = nullptr;
      const int nv = j + 1;
      // cgs2_step (:93-105): h1 = V^T w; w1 = w - V h1; h2 = V^T w1; w2 = w1 - V h2
      if (il && nv <= 16) {  // 3 passes: h1 = V^T w | w1 = w - V h1 with h2 = V^T w1 | w - V h2, ||.||
        LAUNCH(b_launch_dots(d, K.V, nv, K.w, K.mask, K.partials, s));
        LAUNCH(launch_reduce_partials(d, K.partials, nv, K.h1, M + 1, 0, s));
        LAUNCH(b_launch_cgs_dots(d, K.V, nv, K.w, K.h1, M + 1, K.w1, K.mask, K.partials, s));
        LAUNCH(launch_reduce_partials(d, K.partials, nv, K.h2, M + 1, 0, s));
        LAUNCH(b_launch_cgs(d, K.V, nv, K.w1, K.h2, M + 1, K.w, 1, K.mask, K.partials, s));
      } else if (il) {
        LAUNCH(b_launch_dots(d, K.V, nv, K.w, K.mask, K.partials, s));
        LAUNCH(launch_reduce_partials(d, K.partials, nv, K.h1, M + 1, 0, s));
        LAUNCH(b_launch_cgs(d, K.V, nv, K.w, K.h1, M + 1, K.w1, 0, K.mask, nullptr, s));
        LAUNCH(b_launch_dots(d, K.V, nv, K.w1, K.mask, K.partials, s));
        LAUNCH(launch_reduce_partials(d, K.partials, nv, K.h2, M + 1, 0, s));
        LAUNCH(b_launch_cgs(d, K.V, nv, K.w1, K.h2, M + 1, K.w, 1, K.mask, K.partials, s));
      } else {
        LAUNCH((k_dots<<<dim3(G, nb), T, 0, s>>>(K.V, nb, nv, n, K.w, K.mask, K.partials), cudaGetLastError()));
        LAUNCH(launch_reduce_partials(d, K.partials, nv, K.h1, M + 1, 0, s));
        LAUNCH((k_cgs<<<dim3(G, nb), T, 0, s>>>(K.V, nb, nv, n, K.w, K.h1, M + 1, K.w1, 0, K.mask, nullptr),
                cudaGetLastError()));
        LAUNCH((k_dots<<<dim3(G, nb), T, 0, s>>>(K.V, nb, nv, n, K.w1, K.mask, K.partials), cudaGetLastError()));
        LAUNCH(launch_reduce_partials(d, K.partials, nv, K.h2, M + 1, 0, s));
        LAUNCH((k_cgs<<<dim3(G, nb), T, 0, s>>>(K.V, nb, nv, n, K.w1, K.h2, M + 1, K.w, 1, K.mask, K.partials),
                cudaGetLastError()));
      }
      LAUNCH(launch_reduce_partials(d, K.partials, 1, K.nrm, 1, 0, s));
      LAUNCH((k_givens<<<nb, 32, 0, s>>>(K.st, j, M, K.h1, K.h2, K.nrm, K.H, K.cs, K.sn, K.g, K.status,
                                         K.mask, d.scal),
              cudaGetLastError()));
      if ((rc = read_block(dev, K.status, 4 * nb))) return rc;
      bool changed = false;
      for (int q = 0; q < nb; ++q) {
        if (!running[q]) continue;
        const double *stq = dev->pinned + 4 * q;
        if (stq[3] != 0.0) {
          rep[q].iterations = iters[q];
          return fail_nonfinite(q);
        }
        est[q] = stq[0];
        push_hist(q, est[q]);
        iters[q]++;
        jused[q] = j + 1;
        if (stq[1] != 0.0) {  // est <= target or happy breakdown (:184-186)
          running[q] = 0;
          changed = true;
        }
      }
      if (j + 1 < m) {
        if (changed && (rc = upload_mask(dev, running, K.mask))) return rc;
        // V_{j+1} = w / hj1 for the systems still running
        LAUNCH(il ? b_launch_scale(d, K.w, K.V + (size_t)(j + 1) * nbn, K.status + 2, 4, K.mask, s)
                  : (k_scale<<<dim3(G, nb), T, 0, s>>>(K.w, K.V + (size_t)(j + 1) * nbn, n, K.status + 2, 4,
                                                       K.mask),
                     cudaGetLastError()));
      }
    }
    // y = R^{-1} g; x += Z y; r = b - K x; beta = ||r||                      (:189-192)
    if ((rc = upload_mask(dev, jused, K.jused))) return rc;
    LAUNCH((k_solve_upper<<<nb, 32, 0, s>>>(K.H, M, K.g, K.jused, K.yv), cudaGetLastError()));
    LAUNCH(il ? b_launch_update_x(d, K.x, K.Z, K.yv, M + 1, K.jused, s)
              : (k_update_x<<<dim3(G, nb), T, 0, s>>>(K.x, K.Z, nb, n, K.yv, M + 1, K.jused), cudaGetLastError()));
    if ((rc = upload_mask(dev, cycle, K.mask))) return rc;
    d.sys_mask = K.mask;
    if ((rc = dev_spmv(dev, K.x, K.r, b, K.partials))) return rc;
    d.sys_mask = nullptr;
    LAUNCH(launch_reduce_partials(d, K.partials, 1, K.beta, 1, 1, s));
    LAUNCH((k_status<<<1, 64, 0, s>>>(K.status, d.scal, K.beta, nb), cudaGetLastError()));
    if ((rc = read_block(dev, K.status, 4 * nb))) return rc;
    for (int q = 0; q < nb; ++q) {
      if (!cycle[q]) continue;
      beta[q] = dev->pinned[4 * q];
      if (dev->pinned[4 * q + 3] != 0.0) return fail_nonfinite(q);
      restarts[q]++;
      // (:194-198): a stop inside the cycle converges it; otherwise the true residual must
      if (!running[q] || beta[q] <= target[q]) {
        converged[q] = 1;
        active[q] = 0;
      }
    }
  }
  CUDA_TRY(cudaMemcpyAsync(xout, K.x, 8 * nbn, cudaMemcpyDeviceToDevice, s));
  for (int q = 0; q < nb; ++q) {
    rep[q].iterations = iters[q];
    rep[q].precond_applications = iters[q];
    rep[q].converged = converged[q];
    rep[q].restarts = restarts[q];
    rep[q].est_final = est[q];
    rep[q].true_final = beta[q];
  }
  return KKT_OK;
}

}  // namespace kkt
