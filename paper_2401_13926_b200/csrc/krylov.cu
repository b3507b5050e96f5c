// Restarted right-preconditioned FGMRES(m) with CGS2 (krylov.fgmres / cgs2_step,
// krylov.py:93-216) on the device, for nb same-pattern systems at once, with ALL control
// on the device.
//
// Per iteration: z = M v (triangular solves, all running systems in one launch), w = K z
// (SpMV), CGS2 as fused multi-dot / multi-axpy passes, then one control kernel that runs the
// Hessenberg/Givens update of every system (one thread per system), appends the residual
// estimate to the device history and decides, per system, whether it keeps iterating
// (est <= tol*beta0 or happy breakdown stop it, krylov.py:184-186).  Restart cycles, the
// true-residual restart (:189-198), the max_outer budget, per-system non-finite failures
// (:87-90) and the refine trigger (refine.py:113) are decided by device kernels too.
//
// The host never looks at a scalar while the solver runs.  The whole solve is ONE CUDA graph:
//   prologue  [tolerances H2D from pinned memory] -> x = x0 -> r = b - K x, beta -> k_fg_init
//   WHILE (another restart cycle)                                   conditional node
//     k_cycle_begin -> V0 = r / beta
//     IF (any running) iteration 0   ...   IF (any running) iteration m-1   conditional nodes
//     y = R^-1 g -> x += Z y -> r = b - K x, beta -> k_cycle_end
//   epilogue  x_out = x [-> residual statistics of x] -> report block, history, restart
//             pairs D2H into pinned memory
// The control kernels write the condition of the next conditional node with
// cudaGraphSetConditional, so a converged batch skips the remaining iterations without a
// launch.  kkt_dev_step / refine therefore synchronise with the host once per call.
// Host callback operators (the reference's arbitrary LinearOperator) cannot live in a graph:
// that mode replays the same kernels from a host loop that reads the device control flags.
//
// Layouts: V [m+1][nbp][n] (interleaved [n][nbp] per vector on batched handles), Z [m][..];
// per-system control state is [nbp] (structure of arrays), padding systems stay inactive.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "host_util.h"
#include "kernels.cuh"

namespace kkt {

constexpr int FG_THREADS = 1024;  // control kernels: one block, one thread per system

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

// ---- generic operators (single-system handles): identity / callback outputs ----------
// Flags a non-finite entry of v (krylov._check_finite, krylov.py:87-90).
__global__ void k_check_finite(const double *__restrict__ v, int n, unsigned long long *scal) {
  bool bad = false;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (!isfinite(v[i])) bad = true;
  if (bad) atomicOr(&scal[SC_NONFINITE], 1ull);
}

// out = b - y with ||out||^2 block partials [rb] (r = b - K(x) for a non-matrix K).
__global__ void __launch_bounds__(RED_THREADS) k_sub_norm(const double *__restrict__ b,
                                                          const double *__restrict__ y,
                                                          double *__restrict__ out, int n,
                                                          double *__restrict__ partials,
                                                          unsigned long long *scal) {
  __shared__ double sh[32];
  double loc = 0.0;
  bool bad = false;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double yi = y[i];
    if (!isfinite(yi)) bad = true;
    const double o = __dsub_rn(b[i], yi);
    out[i] = o;
    loc = __dadd_rn(loc, __dmul_rn(o, o));
  }
  if (bad) atomicOr(&scal[SC_NONFINITE], 1ull);
  const double t = block_sum<RED_THREADS>(loc, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = t;
}

// ---- device control ------------------------------------------------------------------
// Per-system state (structure of arrays over nbp systems) + the control words.
struct FgCtl {
  double *beta0, *beta, *bnew, *target, *floor_, *est, *hj1, *tolq;
  int *act_in, *active, *running, *cycle, *jused, *iters, *restarts, *converged, *failed, *trig;
  int *vmask;                    // systems whose V_0 = r / beta the cycle start computes
  int *handed;                   // > 0: handed to a helper after that many iterations of its cycle
  int *ctrl;                     // [0..m-1] run iteration j, [m] another cycle, [m+1] cycles run,
                                 // [m+2] iteration bodies run, [m+3] any failure, [m+4] max_outer,
                                 // [m+5] resume at iteration j0 (> 0), [m+6] systems handed off
  unsigned long long *hnd;       // [m+1] conditional handles (IF j, WHILE at m)
  double *hist;                  // [nbp][hcap] est_residual_history
  double *rpair;                 // [nbp][rpcap][2] restart (estimated, true) pairs
  double *repb;                  // [nbp][FG_REP] report block
  double *stats0, *stats1;       // [nbp][5] residual statistics before / after
  unsigned long long *scal;      // the handle's per-system scalar blocks
  double *g, *H, *cs, *sn, *h1, *h2, *nrm;
  int nb, m, M, hcap, rpcap, mode, graph;
  int T;                         // straggler hand-off threshold (running systems; 0 = off)
};

constexpr int FG_REP = 24;  // doubles per system in the report block

__device__ __forceinline__ void fg_set(const FgCtl &c, int slot, int v) {
  c.ctrl[slot] = v;
  if (c.graph) cudaGraphSetConditional(c.hnd[slot], v ? 1u : 0u);
}

__device__ __forceinline__ bool fg_nonfinite(const FgCtl &c, int q) {
  return c.scal[(size_t)q * SCAL_STRIDE + SC_NONFINITE] != 0ull;
}

// Start of fgmres (krylov.py:133-145) / refine_fgmres (refine.py:113): after r = b - K x0 and
// beta = ||r||.  mode 1 (refine): the trigger ||r - K x0||_2 > delta_q ||r||_2 from stats0.
__global__ void __launch_bounds__(FG_THREADS) k_fg_init(FgCtl c) {
  int any = 0, fail = 0;
  for (int q = threadIdx.x; q < c.nb; q += blockDim.x) {
    const int t = c.mode == 1 ? (c.stats0[5 * q] > c.tolq[q] * c.stats0[5 * q + 4] ? 1 : 0)
                              : (c.act_in[q] ? 1 : 0);
    const double b = c.beta[q];
    c.trig[q] = t;
    c.beta0[q] = b;
    c.est[q] = b;
    c.iters[q] = 0;
    c.restarts[q] = 0;
    c.jused[q] = 0;
    c.running[q] = 0;
    c.cycle[q] = 0;
    c.failed[q] = 0;
    c.handed[q] = 0;
    c.converged[q] = t ? 0 : 1;
    c.target[q] = c.tolq[q] * b;
    c.floor_[q] = HAPPY_BREAKDOWN_RTOL * b;
    int act = t;
    if (t) {
      if (c.hcap > 0) c.hist[(size_t)q * c.hcap] = b;
      if (fg_nonfinite(c, q)) {
        c.failed[q] = 1;
        act = 0;
        fail = 1;
      } else if (b == 0.0) {  // (:140-141)
        c.converged[q] = 1;
        act = 0;
      }
    }
    c.active[q] = act;
    any |= act;
  }
  any = __syncthreads_or(any);
  fail = __syncthreads_or(fail);
  if (threadIdx.x == 0) {
    c.ctrl[c.m + 1] = 0;
    c.ctrl[c.m + 2] = 0;
    c.ctrl[c.m + 3] = fail;
    c.ctrl[c.m + 5] = 0;
    c.ctrl[c.m + 6] = 0;
    fg_set(c, c.m, any && c.ctrl[c.m + 4] > 0);
  }
}

// Top of a restart cycle (:147-157): beta <= target converges; else V0 = r / beta follows.
__global__ void __launch_bounds__(FG_THREADS) k_cycle_begin(FgCtl c) {
  int any = 0;
  const int m1 = c.M + 1;
  const int j0 = c.ctrl[c.m + 5];
  if (j0 > 0) {  // a helper resuming a handed-off system inside its cycle, at iteration j0
    for (int q = threadIdx.x; q < c.nb; q += blockDim.x) {
      c.running[q] = c.active[q];
      c.cycle[q] = c.active[q];
      c.vmask[q] = 0;
      c.jused[q] = j0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      c.ctrl[c.m + 5] = 0;
      for (int j = 0; j < c.m; ++j) fg_set(c, j, j == j0);
    }
    return;
  }
  for (int q = threadIdx.x; q < c.nb; q += blockDim.x) {
    int run = 0;
    if (c.active[q]) {
      c.scal[(size_t)q * SCAL_STRIDE + SC_NONFINITE] = 0ull;
      if (c.beta[q] <= c.target[q]) {  // (:148-150)
        c.converged[q] = 1;
        c.active[q] = 0;
      } else {
        run = 1;
        double *gs = c.g + (size_t)q * m1;
        gs[0] = c.beta[q];
        for (int i = 1; i < m1; ++i) gs[i] = 0.0;
        double *Hs = c.H + (size_t)q * m1 * c.M;
        for (int i = 0; i < m1 * c.M; ++i) Hs[i] = 0.0;
      }
    }
    c.running[q] = run;
    c.cycle[q] = run;
    c.vmask[q] = run;
    c.jused[q] = 0;
    any |= run;
  }
  any = __syncthreads_or(any);
  if (threadIdx.x == 0) {
    fg_set(c, 0, any);
    for (int j = 1; j < c.m; ++j) fg_set(c, j, 0);  // set again by iteration j-1 if it runs
  }
}

// Iteration j, after w = K M v_j and CGS2 (h1 + h2, ||w||^2): Hessenberg column j, previous
// rotations, new rotation, estimate, stop test (:164-188) for every running system.
__global__ void __launch_bounds__(FG_THREADS) k_givens(FgCtl c, int j) {
  int any = 0, fail = 0;
  const int m1 = c.M + 1, M = c.M;
  for (int q = threadIdx.x; q < c.nb; q += blockDim.x) {
    if (!c.running[q]) continue;
    if (fg_nonfinite(c, q)) {  // M or K produced NaN/Inf: this system fails (:87-90)
      c.failed[q] = 1;
      c.running[q] = 0;
      c.active[q] = 0;
      c.cycle[q] = 0;
      c.jused[q] = 0;
      fail = 1;
      continue;
    }
    double *Hs = c.H + (size_t)q * m1 * M;
    double *css = c.cs + (size_t)q * m1, *sns = c.sn + (size_t)q * m1, *gs = c.g + (size_t)q * m1;
    for (int i = 0; i <= j; ++i) Hs[i * M + j] = c.h1[(size_t)q * m1 + i] + c.h2[(size_t)q * m1 + i];
    const double hj1 = sqrt(c.nrm[q]);
    Hs[(j + 1) * M + j] = hj1;
    for (int i = 0; i < j; ++i) {
      const double a = Hs[i * M + j], b = Hs[(i + 1) * M + j];
      const double t = __dadd_rn(__dmul_rn(css[i], a), __dmul_rn(sns[i], b));
      Hs[(i + 1) * M + j] = __dadd_rn(__dmul_rn(-sns[i], a), __dmul_rn(css[i], b));
      Hs[i * M + j] = t;
    }
    const double denom = hypot(Hs[j * M + j], Hs[(j + 1) * M + j]);
    css[j] = __ddiv_rn(Hs[j * M + j], denom);
    sns[j] = __ddiv_rn(Hs[(j + 1) * M + j], denom);
    Hs[j * M + j] = denom;
    Hs[(j + 1) * M + j] = 0.0;
    gs[j + 1] = __dmul_rn(-sns[j], gs[j]);
    gs[j] = __dmul_rn(css[j], gs[j]);
    const double est = fabs(gs[j + 1]);
    c.est[q] = est;
    c.hj1[q] = hj1;
    const int it = ++c.iters[q];
    if (it < c.hcap) c.hist[(size_t)q * c.hcap + it] = est;
    c.jused[q] = j + 1;
    if (est <= c.target[q] || hj1 <= c.floor_[q]) c.running[q] = 0;  // (:184-186)
    any |= c.running[q];
  }
  // Straggler hand-off: once at most T systems of the batch still run, the lockstep batch
  // would charge each of their iterations at the whole batch's DAG cost.  They leave the
  // batch here, mid-cycle with their full Krylov state (V_0..j, Z_0..j, H, g, rotations, x),
  // and a single-system helper resumes them at iteration j + 1 (dev_fgmres, resume_handed):
  // the same arithmetic, only another handle.
  __shared__ int s_cnt;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  if (c.T > 0) {
    int mine = 0;
    for (int q = threadIdx.x; q < c.nb; q += blockDim.x) mine += c.running[q];
    if (mine) atomicAdd(&s_cnt, mine);
  }
  __syncthreads();
  const int cnt = s_cnt;
  const bool ho = c.T > 0 && cnt > 0 && cnt <= c.T;
  if (ho) {
    for (int q = threadIdx.x; q < c.nb; q += blockDim.x)
      if (c.running[q]) {
        c.handed[q] = j + 1;
        c.running[q] = 0;
        c.active[q] = 0;
        c.cycle[q] = 0;
        c.jused[q] = 0;  // the batch's cycle end leaves x alone
      }
  }
  any = __syncthreads_or(any);
  fail = __syncthreads_or(fail);
  if (threadIdx.x == 0) {
    c.ctrl[c.m + 2] += 1;
    if (fail) c.ctrl[c.m + 3] = 1;
    if (ho) c.ctrl[c.m + 6] = cnt;
    if (j + 1 < c.m) fg_set(c, j + 1, any && !ho);
  }
}

// End of a cycle (:189-198), after x += Z y and bnew = ||b - K x||: restart pairs, the
// convergence decision, the restart budget.
__global__ void __launch_bounds__(FG_THREADS) k_cycle_end(FgCtl c) {
  int any = 0, fail = 0;
  for (int q = threadIdx.x; q < c.nb; q += blockDim.x) {
    if (c.cycle[q]) {
      if (fg_nonfinite(c, q)) {
        c.failed[q] = 1;
        c.active[q] = 0;
        fail = 1;
      } else {
        const double b = c.bnew[q];
        c.beta[q] = b;
        const int r = c.restarts[q]++;
        if (r < c.rpcap) {
          c.rpair[((size_t)q * c.rpcap + r) * 2] = c.est[q];
          c.rpair[((size_t)q * c.rpcap + r) * 2 + 1] = b;
        }
        if (!c.running[q] || b <= c.target[q]) {  // stopped inside the cycle, or (:196-198)
          c.converged[q] = 1;
          c.active[q] = 0;
        }
      }
    }
    any |= c.active[q];
  }
  any = __syncthreads_or(any);
  fail = __syncthreads_or(fail);
  if (threadIdx.x == 0) {
    const int outer = c.ctrl[c.m + 1] + 1;
    c.ctrl[c.m + 1] = outer;
    if (fail) c.ctrl[c.m + 3] = 1;
    fg_set(c, c.m, any && outer < c.ctrl[c.m + 4]);
  }
}

// Report block: {iterations, converged, restarts, beta0, est_final, true_final, failed,
// triggered, stats0[5], ||K||_inf, stats1[5]} per system.
__global__ void k_fg_report(FgCtl c, int have_stats1) {
  for (int q = threadIdx.x; q < c.nb; q += blockDim.x) {
    double *o = c.repb + (size_t)q * FG_REP;
    o[0] = c.iters[q];
    o[1] = c.converged[q];
    o[2] = c.restarts[q];
    o[3] = c.beta0[q];
    o[4] = c.est[q];
    o[5] = c.trig[q] ? c.beta[q] : c.beta0[q];
    o[6] = c.failed[q];
    o[7] = c.trig[q];
    for (int i = 0; i < 5; ++i) o[8 + i] = c.mode == 1 ? c.stats0[5 * q + i] : 0.0;
    o[13] = __longlong_as_double((long long)c.scal[(size_t)q * SCAL_STRIDE + SC_OPNORM]);
    for (int i = 0; i < 5; ++i) o[14 + i] = have_stats1 ? c.stats1[5 * q + i] : 0.0;
    o[19] = c.handed[q];
  }
}

// Unpack the host-staged inputs: in = {tolq[nbp], act_in[nbp] (as doubles), max_outer}.
__global__ void k_unpack_inputs(const double *in, int nbp, int *act_in, int *ctrl, int m) {
  for (int q = threadIdx.x; q < nbp; q += blockDim.x) act_in[q] = in[nbp + q] != 0.0;
  if (threadIdx.x == 0) ctrl[m + 4] = (int)in[2 * nbp];
}

__global__ void k_clear_nonfinite(unsigned long long *scal, int nb) {
  for (int q = threadIdx.x; q < nb; q += blockDim.x) scal[(size_t)q * SCAL_STRIDE + SC_NONFINITE] = 0ull;
}

// ---- straggler hand-off (batched handle -> single-system helper) ------------------------
// dst[i] = src[i * stride + off]: one system's column of an interleaved [count][stride] array
__global__ void k_gather_col(double *__restrict__ dst, const double *__restrict__ src, int64_t count,
                             int stride, int off) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i * stride + off];
}
__global__ void k_scatter_col(double *__restrict__ dst, const double *__restrict__ src, int64_t count,
                              int stride, int off) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    dst[i * stride + off] = src[i];
}

// The per-system control state of system q of the batch (src) -> the helper's system 0 (dst):
// everything k_givens / k_cycle_end / k_fg_report read, the Hessenberg / rotation state of the
// open cycle, the histories, the scalar block; resume at iteration j0 of the current cycle.
__global__ void k_handoff_state(FgCtl src, FgCtl dst, int q, int j0, const double *__restrict__ sbeta,
                                double *__restrict__ dbeta) {
  const int m1 = src.M + 1;
  for (int i = threadIdx.x; i < m1 * src.M; i += blockDim.x) dst.H[i] = src.H[(size_t)q * m1 * src.M + i];
  for (int i = threadIdx.x; i < m1; i += blockDim.x) {
    dst.g[i] = src.g[(size_t)q * m1 + i];
    dst.cs[i] = src.cs[(size_t)q * m1 + i];
    dst.sn[i] = src.sn[(size_t)q * m1 + i];
  }
  for (int i = threadIdx.x; i < min(src.hcap, dst.hcap); i += blockDim.x)
    dst.hist[i] = src.hist[(size_t)q * src.hcap + i];
  for (int i = threadIdx.x; i < 2 * min(src.rpcap, dst.rpcap); i += blockDim.x)
    dst.rpair[i] = src.rpair[(size_t)q * src.rpcap * 2 + i];
  for (int i = threadIdx.x; i < SCAL_STRIDE; i += blockDim.x)
    dst.scal[i] = src.scal[(size_t)q * SCAL_STRIDE + i];
  if (threadIdx.x == 0) {
    dst.beta0[0] = src.beta0[q];
    dbeta[0] = sbeta[q];
    dst.target[0] = src.target[q];
    dst.floor_[0] = src.floor_[q];
    dst.est[0] = src.est[q];
    dst.hj1[0] = src.hj1[q];
    dst.iters[0] = src.iters[q];
    dst.restarts[0] = src.restarts[q];
    dst.trig[0] = src.trig[q];
    dst.converged[0] = 0;
    dst.failed[0] = 0;
    dst.handed[0] = 0;
    dst.active[0] = 1;
    dst.running[0] = 1;
    dst.cycle[0] = 1;
    dst.jused[0] = j0;
    for (int i = 0; i < 5; ++i) dst.stats0[i] = src.stats0[5 * q + i];
    // cycles completed: the batch's count minus the open cycle (its end ran without q)
    dst.ctrl[dst.m + 1] = src.ctrl[src.m + 1] - 1;
    dst.ctrl[dst.m + 5] = j0;
  }
}

// Helper prologue: V_j0 = w / h_{j0,j0-1} (the scale the batch skipped for the handed system),
// the first cycle's WHILE condition.
__global__ void __launch_bounds__(RED_THREADS) k_resume_begin(FgCtl c, double *__restrict__ V,
                                                              const double *__restrict__ w, int n) {
  const int j0 = c.ctrl[c.m + 5];
  if (j0 < c.m) {
    const double dv = c.hj1[0];
    double *vj = V + (size_t)j0 * n;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
      vj[i] = __ddiv_rn(w[i], dv);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    c.ctrl[c.m + 2] = 0;
    c.ctrl[c.m + 3] = 0;
    c.ctrl[c.m + 6] = 0;
    fg_set(c, c.m, 1);
  }
}

// ---- workspace -------------------------------------------------------------------------
static void free_graphs(Krylov *K) {
  for (FgGraph &g : K->graphs) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    if (g.graph) cudaGraphDestroy(g.graph);
  }
  K->graphs.clear();
}

void free_krylov(Device *dev) {
  if (dev->kry) {
    free_graphs(dev->kry);
    cudaFree(dev->kry->mem);
    cudaFree(dev->kry->cmem);
    cudaFreeHost(dev->kry->pin);
    if (dev->kry->cb_pin) cudaFreeHost(dev->kry->cb_pin);
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
  bytes += 2 * align_up(8 * nb + 64);
  bytes += align_up(8 * (m + 2) * rb * nb + 1);
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
  K->partials = carve<double>(cur, (m + 2) * rb * nb);
  free_krylov(dev);
  dev->kry = K;
  return KKT_OK;
}

// Grow the workspace BEFORE a caller stages vectors in it (K.sr / sx0 / sx): growing frees
// the old one.
int ensure_krylov(Device *dev, int m) {
  if (m < 1) return set_error(KKT_ERR_BAD_ARG, "restart length m must be >= 1");
  if (m > 62) return set_error(KKT_ERR_BAD_ARG, "restart length m must be <= 62");
  if (dev->kry && dev->kry->m >= m) return KKT_OK;
  return alloc_krylov(dev, m);
}

// Control state sized for (m, max_outer); reallocation drops the cached graphs.
static int ensure_control(Device *dev, int m, int max_outer) {
  Krylov &K = *dev->kry;
  const int hcap = max_outer * m + 1, rpcap = std::max(max_outer, 1);
  if (K.cmem && K.c_hcap >= hcap && K.c_rpcap >= rpcap && K.c_m >= m) return KKT_OK;
  free_graphs(&K);
  if (K.cmem) cudaFree(K.cmem);
  if (K.pin) cudaFreeHost(K.pin);
  K.cmem = nullptr;
  K.pin = nullptr;
  const size_t nb = (size_t)dev->d.nbp;
  K.c_hcap = std::max(hcap, K.c_hcap);
  K.c_rpcap = std::max(rpcap, K.c_rpcap);
  K.c_m = std::max(m, K.c_m);
  const size_t out_doubles = nb * FG_REP + nb * K.c_hcap + nb * K.c_rpcap * 2 + 16;
  const size_t in_doubles = nb * 2 + 8;
  size_t bytes = 6 * align_up(8 * nb + 64) + 12 * align_up(4 * nb + 64) + align_up(4 * (K.c_m + 8)) +
                 align_up(8 * (K.c_m + 1)) + align_up(8 * out_doubles) + 2 * align_up(8 * 5 * nb + 64) +
                 align_up(8 * in_doubles);
  CUDA_TRY(cudaMalloc(&K.cmem, bytes));
  CUDA_TRY(cudaMemsetAsync(K.cmem, 0, bytes, dev->stream));
  // pinned: [outputs][inputs][control words]
  K.pin_bytes = 8 * (out_doubles + in_doubles) + 4 * (K.c_m + 8) + 64;
  CUDA_TRY(cudaMallocHost(&K.pin, K.pin_bytes));
  std::memset(K.pin, 0, K.pin_bytes);
  K.pin_ctrl = reinterpret_cast<int *>(K.pin + out_doubles + in_doubles);
  char *cur = (char *)K.cmem;
  FgBufs &B = K.fb;
  B.beta0 = carve<double>(cur, nb + 8);
  B.bnew = carve<double>(cur, nb + 8);
  B.target = carve<double>(cur, nb + 8);
  B.floor_ = carve<double>(cur, nb + 8);
  B.est = carve<double>(cur, nb + 8);
  B.hj1 = carve<double>(cur, nb + 8);
  B.act_in = carve<int>(cur, nb + 16);
  B.active = carve<int>(cur, nb + 16);
  B.running = carve<int>(cur, nb + 16);
  B.cycle = carve<int>(cur, nb + 16);
  B.jused = carve<int>(cur, nb + 16);
  B.iters = carve<int>(cur, nb + 16);
  B.restarts = carve<int>(cur, nb + 16);
  B.converged = carve<int>(cur, nb + 16);
  B.failed = carve<int>(cur, nb + 16);
  B.trig = carve<int>(cur, nb + 16);
  B.handed = carve<int>(cur, nb + 16);
  B.vmask = carve<int>(cur, nb + 16);
  B.ctrl = carve<int>(cur, K.c_m + 8);
  B.hnd = carve<unsigned long long>(cur, K.c_m + 1);
  B.out = carve<double>(cur, out_doubles);
  B.stats0 = carve<double>(cur, 5 * nb + 8);
  B.stats1 = carve<double>(cur, 5 * nb + 8);
  B.in = carve<double>(cur, in_doubles);
  B.out_doubles = out_doubles;
  B.in_doubles = in_doubles;
  return KKT_OK;
}

// ---- one FGMRES solve -------------------------------------------------------------------
namespace {

struct Call {
  const double *b, *x0;
  double *xout;
  int m, max_outer, mode, want_after, mgs;
  const kkt_linop *opK, *opM;  // nullptr = the handle's operator / LU factors
  int resume = 0;  // a helper continuing a handed-off system (state staged by resume_handed)
  int T = 0;       // straggler hand-off threshold of a batched handle
};

int op_kind(const kkt_linop *op) { return op ? op->kind : KKT_OP_HANDLE; }

struct Runner {
  Device *dev;
  Krylov &K;
  const Call &C;
  FgCtl c;
  cudaStream_t s;
  int nbp, n;
  size_t nbn;
  bool il;

  Runner(Device *d, const Call &call) : dev(d), K(*d->kry), C(call), s(d->stream) {
    nbp = dev->d.nbp;
    n = dev->d.n;
    nbn = (size_t)nbp * n;
    il = nbp > 1;
    const FgBufs &B = K.fb;
    c.beta0 = B.beta0;
    c.beta = K.beta;
    c.bnew = B.bnew;
    c.target = B.target;
    c.floor_ = B.floor_;
    c.est = B.est;
    c.hj1 = B.hj1;
    c.tolq = B.in;  // [nbp] tolerances (then the act_in flags and max_outer, k_unpack_inputs)
    c.act_in = B.act_in;
    c.active = B.active;
    c.running = B.running;
    c.cycle = B.cycle;
    c.jused = B.jused;
    c.iters = B.iters;
    c.restarts = B.restarts;
    c.converged = B.converged;
    c.failed = B.failed;
    c.trig = B.trig;
    c.handed = B.handed;
    c.vmask = B.vmask;
    c.ctrl = B.ctrl;
    c.hnd = B.hnd;
    c.repb = B.out;
    c.hist = B.out + (size_t)nbp * FG_REP;
    c.rpair = c.hist + (size_t)nbp * K.c_hcap;
    c.stats0 = B.stats0;
    c.stats1 = B.stats1;
    c.scal = dev->d.scal;
    c.g = K.g;
    c.H = K.H;
    c.cs = K.cs;
    c.sn = K.sn;
    c.h1 = K.h1;
    c.h2 = K.h2;
    c.nrm = K.nrm;
    c.nb = dev->d.nb;
    c.m = C.m;
    c.M = K.m;
    c.hcap = K.c_hcap;
    c.rpcap = K.c_rpcap;
    c.mode = C.mode;
    c.graph = 0;
    c.T = C.T;
  }

  // ---- operator applications (M: LU solve / identity / callback; K: SpMV / ...) ----
  int apply_M(const double *in, double *out, const int *mask) {
    const kkt_linop *op = C.opM;
    switch (op_kind(op)) {
      case KKT_OP_HANDLE: {
        dev->d.sys_mask = mask;
        int rc = dev_solve(dev, in, out);
        dev->d.sys_mask = nullptr;
        return rc;
      }
      case KKT_OP_MATRIX:
        return op_matrix(op, in, out, nullptr, nullptr);
      case KKT_OP_IDENTITY:
        CUDA_TRY(cudaMemcpyAsync(out, in, 8 * (size_t)n, cudaMemcpyDeviceToDevice, s));
        LAUNCH((k_check_finite<<<dev->d.rb, RED_THREADS, 0, s>>>(out, n, dev->d.scal), cudaGetLastError()));
        return KKT_OK;
      default:
        return callback(op, in, out, nullptr, nullptr);
    }
  }

  // out = K in, or out = bsub - K in with ||out||^2 partials
  int apply_K(const double *in, double *out, const double *bsub, double *partials, const int *mask) {
    const kkt_linop *op = C.opK;
    switch (op_kind(op)) {
      case KKT_OP_HANDLE: {
        dev->d.sys_mask = mask;
        int rc = dev_spmv(dev, in, out, bsub, partials);
        dev->d.sys_mask = nullptr;
        return rc;
      }
      case KKT_OP_MATRIX:
        return op_matrix(op, in, out, bsub, partials);
      case KKT_OP_IDENTITY:
        if (bsub) {
          LAUNCH((k_sub_norm<<<dev->d.rb, RED_THREADS, 0, s>>>(bsub, in, out, n, partials, dev->d.scal),
                  cudaGetLastError()));
          return KKT_OK;
        }
        CUDA_TRY(cudaMemcpyAsync(out, in, 8 * (size_t)n, cudaMemcpyDeviceToDevice, s));
        return KKT_OK;
      default:
        return callback(op, in, out, bsub, partials);
    }
  }

  int op_matrix(const kkt_linop *op, const double *in, double *out, const double *bsub, double *partials) {
    const Operator *A = reinterpret_cast<const Operator *>(op->matrix);
    DevPlan od = A->d;  // the bare operator's pattern/values, this handle's flags + partials
    od.scal = dev->d.scal;
    od.rb = dev->d.rb;
    LAUNCH(launch_spmv(od, in, out, bsub, partials, s));
    return KKT_OK;
  }

  // Host operator (the reference's LinearOperator callback on numpy vectors): in is copied
  // to a pinned host buffer, apply() fills the other one, the result goes back to out.
  int callback(const kkt_linop *op, const double *in, double *out, const double *bsub, double *partials) {
    if (!K.cb_pin) CUDA_TRY(cudaMallocHost(&K.cb_pin, 16 * (size_t)n + 64));
    double *hin = K.cb_pin, *hout = K.cb_pin + n;
    CUDA_TRY(cudaMemcpyAsync(hin, in, 8 * (size_t)n, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (op->apply(op->user, hin, hout) != 0) return set_error(KKT_ERR_CALLBACK, "operator callback failed");
    CUDA_TRY(cudaMemcpyAsync(out, hout, 8 * (size_t)n, cudaMemcpyHostToDevice, s));
    if (bsub) {
      LAUNCH((k_sub_norm<<<dev->d.rb, RED_THREADS, 0, s>>>(bsub, out, out, n, partials, dev->d.scal),
              cudaGetLastError()));
    } else {
      LAUNCH((k_check_finite<<<dev->d.rb, RED_THREADS, 0, s>>>(out, n, dev->d.scal), cudaGetLastError()));
    }
    // the host buffers are reused by the next call: wait for the upload
    CUDA_TRY(cudaStreamSynchronize(s));
    return KKT_OK;
  }

  // ---- segments ----
  int prologue() {
    DevPlan &d = dev->d;
    const FgBufs &B = K.fb;
    // per-system tolerances / active flags staged by the host in pinned memory
    CUDA_TRY(cudaMemcpyAsync(B.in, K.pin + B.out_doubles, 8 * B.in_doubles, cudaMemcpyHostToDevice, s));
    LAUNCH((k_unpack_inputs<<<1, 256, 0, s>>>(B.in, nbp, B.act_in, B.ctrl, C.m), cudaGetLastError()));
    if (C.resume) {  // the state is staged (resume_handed): V_j0 = w / h_{j0,j0-1}, then the cycle
      LAUNCH((k_resume_begin<<<d.rb, RED_THREADS, 0, s>>>(c, K.V, K.w, n), cudaGetLastError()));
      return KKT_OK;
    }
    LAUNCH((k_clear_nonfinite<<<1, 256, 0, s>>>(d.scal, d.nb), cudaGetLastError()));
    if (C.mode == 1) {  // refine: statistics of (r, x0) decide the trigger (refine.py:113)
      LAUNCH(il ? b_launch_resid_stats(d, C.b, C.x0, d.partials, B.stats0, s)
                : launch_resid_stats(d, C.b, C.x0, d.partials, B.stats0, s));
    }
    CUDA_TRY(cudaMemcpyAsync(K.x, C.x0, 8 * nbn, cudaMemcpyDeviceToDevice, s));
    int rc = apply_K(K.x, K.r, C.b, K.partials, nullptr);  // r = b - K x; beta0 = ||r|| (:133-134)
    if (rc) return rc;
    LAUNCH(launch_reduce_partials(d, K.partials, 1, K.beta, 1, 1, s));
    LAUNCH((k_fg_init<<<1, FG_THREADS, 0, s>>>(c), cudaGetLastError()));
    return KKT_OK;
  }

  int cycle_begin() {
    LAUNCH((k_cycle_begin<<<1, FG_THREADS, 0, s>>>(c), cudaGetLastError()));
    LAUNCH(scale(K.r, K.V, K.beta, 1, c.vmask));  // V0 = r / beta (a division, :151)
    return KKT_OK;
  }

  cudaError_t scale(const double *in, double *out, const double *den, int dstride, const int *mask) {
    if (il) return b_launch_scale(dev->d, in, out, den, dstride, mask, s);
    k_scale<<<dim3(dev->d.rb, nbp), RED_THREADS, 0, s>>>(in, out, n, den, dstride, mask);
    return cudaGetLastError();
  }

  int iteration(int j) {
    DevPlan &d = dev->d;
    const int M = K.m;
    double *Vj = K.V + (size_t)j * nbn;
    double *Zj = K.Z + (size_t)j * nbn;
    int rc = apply_M(Vj, Zj, c.running);  // z = M(V_j)   :161
    if (rc) return rc;
    if ((rc = apply_K(Zj, K.w, nullptr, nullptr, c.running))) return rc;  // w = K z  :163
    const int nv = j + 1;
    const int *mask = c.running;
    if (C.mgs) {  // _mgs_step (krylov.py:108-114): h_i = v_i . w; w -= h_i v_i, one basis vector at a time
      CUDA_TRY(cudaMemsetAsync(K.h2, 0, 8 * (size_t)nbp * (M + 1), s));
      for (int i = 0; i < nv; ++i) {
        const double *Vi = K.V + (size_t)i * nbn;
        const int last = i + 1 == nv;
        if (il) {
          LAUNCH(b_launch_dots(d, Vi, 1, K.w, mask, K.partials, s));
          LAUNCH(launch_reduce_partials(d, K.partials, 1, K.h1 + i, M + 1, 0, s));
          LAUNCH(b_launch_cgs(d, Vi, 1, K.w, K.h1 + i, M + 1, K.w, last, mask, last ? K.partials : nullptr, s));
        } else {
          LAUNCH((k_dots<<<dim3(d.rb, nbp), RED_THREADS, 0, s>>>(Vi, nbp, 1, n, K.w, mask, K.partials),
                  cudaGetLastError()));
          LAUNCH(launch_reduce_partials(d, K.partials, 1, K.h1 + i, M + 1, 0, s));
          LAUNCH((k_cgs<<<dim3(d.rb, nbp), RED_THREADS, 0, s>>>(Vi, nbp, 1, n, K.w, K.h1 + i, M + 1, K.w, last,
                                                                 mask, last ? K.partials : nullptr),
                  cudaGetLastError()));
        }
      }
    } else
    // cgs2_step (:93-105): h1 = V^T w; w1 = w - V h1; h2 = V^T w1; w2 = w1 - V h2
    if (il && nv <= 16) {  // 3 passes: h1 = V^T w | w1 = w - V h1 with h2 = V^T w1 | w - V h2, ||.||
      LAUNCH(b_launch_dots(d, K.V, nv, K.w, mask, K.partials, s));
      LAUNCH(launch_reduce_partials(d, K.partials, nv, K.h1, M + 1, 0, s));
      LAUNCH(b_launch_cgs_dots(d, K.V, nv, K.w, K.h1, M + 1, K.w1, mask, K.partials, s));
      LAUNCH(launch_reduce_partials(d, K.partials, nv, K.h2, M + 1, 0, s));
      LAUNCH(b_launch_cgs(d, K.V, nv, K.w1, K.h2, M + 1, K.w, 1, mask, K.partials, s));
    } else if (il) {
      LAUNCH(b_launch_dots(d, K.V, nv, K.w, mask, K.partials, s));
      LAUNCH(launch_reduce_partials(d, K.partials, nv, K.h1, M + 1, 0, s));
      LAUNCH(b_launch_cgs(d, K.V, nv, K.w, K.h1, M + 1, K.w1, 0, mask, nullptr, s));
      LAUNCH(b_launch_dots(d, K.V, nv, K.w1, mask, K.partials, s));
      LAUNCH(launch_reduce_partials(d, K.partials, nv, K.h2, M + 1, 0, s));
      LAUNCH(b_launch_cgs(d, K.V, nv, K.w1, K.h2, M + 1, K.w, 1, mask, K.partials, s));
    } else {
      const int G = d.rb, T = RED_THREADS, nb = nbp;
      LAUNCH((k_dots<<<dim3(G, nb), T, 0, s>>>(K.V, nb, nv, n, K.w, mask, K.partials), cudaGetLastError()));
      LAUNCH(launch_reduce_partials(d, K.partials, nv, K.h1, M + 1, 0, s));
      LAUNCH((k_cgs<<<dim3(G, nb), T, 0, s>>>(K.V, nb, nv, n, K.w, K.h1, M + 1, K.w1, 0, mask, nullptr),
              cudaGetLastError()));
      LAUNCH((k_dots<<<dim3(G, nb), T, 0, s>>>(K.V, nb, nv, n, K.w1, mask, K.partials), cudaGetLastError()));
      LAUNCH(launch_reduce_partials(d, K.partials, nv, K.h2, M + 1, 0, s));
      LAUNCH((k_cgs<<<dim3(G, nb), T, 0, s>>>(K.V, nb, nv, n, K.w1, K.h2, M + 1, K.w, 1, mask, K.partials),
              cudaGetLastError()));
    }
    LAUNCH(launch_reduce_partials(d, K.partials, 1, K.nrm, 1, 0, s));
    LAUNCH((k_givens<<<1, FG_THREADS, 0, s>>>(c, j), cudaGetLastError()));
    if (j + 1 < C.m)  // V_{j+1} = w / hj1 for the systems still running (:188)
      LAUNCH(scale(K.w, K.V + (size_t)(j + 1) * nbn, c.hj1, 1, c.running));
    return KKT_OK;
  }

  int cycle_end() {
    DevPlan &d = dev->d;
    const int M = K.m;
    // y = R^{-1} g; x += Z y; r = b - K x; beta = ||r||                      (:189-192)
    LAUNCH((k_solve_upper<<<nbp, 32, 0, s>>>(K.H, M, K.g, c.jused, K.yv), cudaGetLastError()));
    LAUNCH(il ? b_launch_update_x(d, K.x, K.Z, K.yv, M + 1, c.jused, s)
              : (k_update_x<<<dim3(d.rb, nbp), RED_THREADS, 0, s>>>(K.x, K.Z, nbp, n, K.yv, M + 1, c.jused),
                 cudaGetLastError()));
    int rc = apply_K(K.x, K.r, C.b, K.partials, c.cycle);
    if (rc) return rc;
    LAUNCH(launch_reduce_partials(d, K.partials, 1, c.bnew, 1, 1, s));
    LAUNCH((k_cycle_end<<<1, FG_THREADS, 0, s>>>(c), cudaGetLastError()));
    return KKT_OK;
  }

  int epilogue() {
    DevPlan &d = dev->d;
    const FgBufs &B = K.fb;
    CUDA_TRY(cudaMemcpyAsync(C.xout, K.x, 8 * nbn, cudaMemcpyDeviceToDevice, s));
    if (C.want_after)
      LAUNCH(il ? b_launch_resid_stats(d, C.b, C.xout, d.partials, B.stats1, s)
                : launch_resid_stats(d, C.b, C.xout, d.partials, B.stats1, s));
    LAUNCH((k_fg_report<<<1, 256, 0, s>>>(c, C.want_after), cudaGetLastError()));
    CUDA_TRY(cudaMemcpyAsync(K.pin, B.out, 8 * B.out_doubles, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(K.pin_ctrl, B.ctrl, 4 * (K.c_m + 8), cudaMemcpyDeviceToHost, s));
    return KKT_OK;
  }

  // ---- host-stepped control (callback operators; KKT_FG_HOST_LOOP) ----
  int read_ctrl() {
    CUDA_TRY(cudaMemcpyAsync(K.pin_ctrl, K.fb.ctrl, 4 * (K.c_m + 8), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return KKT_OK;
  }

  int run_host() {
    int rc = prologue();
    if (rc) return rc;
    if ((rc = read_ctrl())) return rc;
    while (K.pin_ctrl[C.m]) {
      if ((rc = cycle_begin()) || (rc = read_ctrl())) return rc;
      for (int j = 0; j < C.m && K.pin_ctrl[j]; ++j)
        if ((rc = iteration(j)) || (rc = read_ctrl())) return rc;
      if ((rc = cycle_end()) || (rc = read_ctrl())) return rc;
    }
    if ((rc = epilogue())) return rc;
    CUDA_TRY(cudaStreamSynchronize(s));
    return KKT_OK;
  }

  // ---- graph mode ----
  // Capture the stream's work issued by f() into graph g after the nodes deps.
  template <typename F>
  int capture(cudaGraph_t g, const cudaGraphNode_t *deps, size_t ndeps, F f,
              std::vector<cudaGraphNode_t> *frontier) {
    CUDA_TRY(cudaStreamBeginCaptureToGraph(s, g, deps, nullptr, ndeps, cudaStreamCaptureModeRelaxed));
    int rc = f();
    if (rc == KKT_OK && frontier) {
      cudaStreamCaptureStatus st;
      const cudaGraphNode_t *fd = nullptr;
      size_t nf = 0;
      cudaError_t e = cudaStreamGetCaptureInfo(s, &st, nullptr, nullptr, &fd, &nf);
      if (e != cudaSuccess) rc = set_error(KKT_ERR_CUDA, cudaGetErrorString(e));
      else frontier->assign(fd, fd + nf);
    }
    cudaGraph_t out = nullptr;
    cudaError_t e = cudaStreamEndCapture(s, &out);
    if (rc) return rc;
    if (e != cudaSuccess) return set_error(KKT_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    return KKT_OK;
  }

  int add_cond(cudaGraph_t g, const std::vector<cudaGraphNode_t> &deps, cudaGraphConditionalHandle h,
               cudaGraphConditionalNodeType type, cudaGraphNode_t *node, cudaGraph_t *body) {
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = type;
    p.conditional.size = 1;
    CUDA_TRY(cudaGraphAddNode(node, g, deps.data(), deps.size(), &p));
    *body = p.conditional.phGraph_out[0];
    return KKT_OK;
  }

  int build_graph(FgGraph &G) {
    c.graph = 1;
    const long long l0 = dev->launches;
    cudaGraph_t g = nullptr;
    CUDA_TRY(cudaGraphCreate(&g, 0));
    G.graph = g;
    std::vector<cudaGraphConditionalHandle> h(C.m + 1);
    CUDA_TRY(cudaGraphConditionalHandleCreate(&h[C.m], g, 0, cudaGraphCondAssignDefault));
    std::vector<cudaGraphNode_t> fr;
    int rc = capture(g, nullptr, 0, [&] { return prologue(); }, &fr);
    if (rc) return rc;
    G.l_pro = dev->launches - l0;
    cudaGraphNode_t wn;
    cudaGraph_t body;
    if ((rc = add_cond(g, fr, h[C.m], cudaGraphCondTypeWhile, &wn, &body))) return rc;
    // the restart cycle
    for (int j = 0; j < C.m; ++j) CUDA_TRY(cudaGraphConditionalHandleCreate(&h[j], body, 0, cudaGraphCondAssignDefault));
    if ((rc = capture(body, nullptr, 0, [&] { return cycle_begin(); }, &fr))) return rc;
    for (int j = 0; j < C.m; ++j) {
      cudaGraphNode_t in;
      cudaGraph_t ib;
      if ((rc = add_cond(body, fr, h[j], cudaGraphCondTypeIf, &in, &ib))) return rc;
      const long long li = dev->launches;
      if ((rc = capture(ib, nullptr, 0, [&] { return iteration(j); }, nullptr))) return rc;
      if (j == 0) G.l_iter = dev->launches - li;
      fr.assign(1, in);
    }
    const long long l2 = dev->launches;
    if ((rc = capture(body, fr.data(), fr.size(), [&] { return cycle_end(); }, nullptr))) return rc;
    G.l_cyc = (dev->launches - l2) + 2;
    const cudaGraphNode_t wdep[1] = {wn};
    if ((rc = capture(g, wdep, 1, [&] { return epilogue(); }, nullptr))) return rc;
    G.l_epi = 2 + (C.want_after ? 1 : 0);
    // the handles the control kernels set
    std::vector<unsigned long long> hv(h.begin(), h.end());
    CUDA_TRY(cudaMemcpyAsync(K.fb.hnd, hv.data(), 8 * hv.size(), cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    CUDA_TRY(cudaGraphInstantiate(&G.exec, g, 0));
    dev->launches = l0;  // capture issued nothing; launches are counted per execution
    return KKT_OK;
  }
};

// Everything a captured graph depends on besides the (fixed) workspace pointers.
void graph_key(const Device *dev, const Call &C, FgGraph &k) {
  k.b = C.b;
  k.x0 = C.x0;
  k.xout = C.xout;
  k.m = C.m;
  k.mode = C.mode;
  k.want_after = C.want_after;
  k.mgs = C.mgs;
  k.resume = C.resume;
  k.T = C.T;
  k.plan = dev->d;
  k.plan.sys_mask = nullptr;
}

bool same_key(const FgGraph &a, const FgGraph &b) {
  return a.b == b.b && a.x0 == b.x0 && a.xout == b.xout && a.m == b.m && a.mode == b.mode &&
         a.want_after == b.want_after && a.mgs == b.mgs && a.resume == b.resume && a.T == b.T && std::memcmp(&a.plan, &b.plan, sizeof(DevPlan)) == 0;
}

}  // namespace

// Running systems at or below which a batch hands its stragglers to single-system helpers
// (KKT_HANDOFF=T overrides; 0 disables).  A helper's iteration costs a single system's DAG
// latency instead of the whole batch's (10k: ~1.4 ms vs ~4.5 ms at B = 64).
static int handoff_threshold(int nb) {
  if (const char *e = std::getenv("KKT_HANDOFF")) return std::max(0, std::atoi(e));
  return nb >= 16 ? std::min(4, nb / 16) : 0;
}

// Create a batched handle's straggler helpers up front (kkt_dev_create), so the first
// hand-off does not pay for their allocation.
int prepare_helpers(Device *dev) {
  const int T = dev->d.nbp > 1 ? handoff_threshold(dev->d.nb) : 0;
  while ((int)dev->helpers.size() < T) {
    Device *h = nullptr;
    int rc = create_like(dev, 1, h);
    if (rc) return rc;
    dev->helpers.push_back(h);
    if ((rc = ensure_control(h, h->restart_m, 10))) return rc;
  }
  return KKT_OK;
}

// The cached graph for (handle, call), captured on first use.
static int get_graph(Device *dev, Runner &R, const Call &C, FgGraph *&G) {
  Krylov &K = *dev->kry;
  FgGraph key;
  graph_key(dev, C, key);
  G = nullptr;
  for (FgGraph &g : K.graphs)
    if (same_key(g, key)) G = &g;
  if (G) return KKT_OK;
  if (K.graphs.size() >= 6) {
    FgGraph &old = K.graphs.front();
    if (old.exec) cudaGraphExecDestroy(old.exec);
    if (old.graph) cudaGraphDestroy(old.graph);
    K.graphs.erase(K.graphs.begin());
  }
  K.graphs.push_back(key);
  G = &K.graphs.back();
  int rc = R.build_graph(*G);
  if (rc) {
    if (G->exec) cudaGraphExecDestroy(G->exec);
    if (G->graph) cudaGraphDestroy(G->graph);
    K.graphs.pop_back();
    G = nullptr;
  }
  return rc;
}

// Resume every handed-off system q of the batch on its own single-system helper handle, all
// helpers concurrently on their own streams: gather q's factors, operator values, scalar block
// and open Krylov cycle (V_0..j0-1, w, Z_0..j0-1, x, b, H, g, rotations, counters, histories)
// out of the interleaved layout, run the helper's resume graph (the rest of q's FGMRES), and
// scatter its x back into the batch's solution.  Everything after the batch's own graph; one
// host synchronisation for all helpers.
static int resume_handed(Device *dev, Runner &R, const Call &C, const std::vector<int> &handed) {
  Krylov &K = *dev->kry;
  const DevPlan &d = dev->d;
  const int nbp = d.nbp, n = d.n;
  const size_t nbn = (size_t)nbp * n;
  const cudaStream_t s = dev->stream;
  while (dev->helpers.size() < handed.size()) {
    Device *h = nullptr;
    int rc = create_like(dev, 1, h);
    if (rc) return rc;
    dev->helpers.push_back(h);
  }
  if (!dev->ev_h) CUDA_TRY(cudaEventCreateWithFlags(&dev->ev_h, cudaEventDisableTiming));
  // Concurrent by default: every helper on its own stream.  The single-system grid solve is a
  // persistent sync-free kernel (its CTAs wait on each other), so each helper's grid is cut to
  // a 1/T share of the GPU's resident-CTA capacity: the T persistent grids together never
  // exceed it and are co-resident whatever the interleaving (the single solve is as fast with
  // 296 CTAs as with 1184: 1.26 ms at 10k).  KKT_HANDOFF_CONCURRENT=0: one after the other on
  // the batch's stream with full grids.
  const char *ce = std::getenv("KKT_HANDOFF_CONCURRENT");
  const bool concurrent = !ce || std::atoi(ce) != 0;
  // the batch's graph is complete (synchronised): helpers may read its state
  const int G = 2 * dev->sm_count;
  auto gather = [&](cudaStream_t st, double *dst, const double *srcp, int64_t cnt, int q) -> cudaError_t {
    if (cnt <= 0) return cudaSuccess;
    k_gather_col<<<G, 256, 0, st>>>(dst, srcp, cnt, nbp, q);
    return cudaGetLastError();
  };
  std::vector<FgGraph *> graphs(handed.size(), nullptr);
  std::vector<Call> calls(handed.size(), C);
  for (size_t i = 0; i < handed.size(); ++i) {
    Device *h = dev->helpers[i];
    const int q = handed[i];
    const int j0 = (int)K.pin[(size_t)q * FG_REP + 19];
    int rc;
    if (!h->kry || h->kry->m != K.m) {
      if ((rc = alloc_krylov(h, K.m))) return rc;
    }
    if ((rc = ensure_control(h, C.m, std::max(C.max_outer, 1)))) return rc;
    Krylov &HK = *h->kry;
    DevPlan &hd = h->d;
    hd.sym_lower = d.sym_lower;
    hd.has_lower = d.has_lower;
    const cudaStream_t hs = concurrent ? h->stream : s;
    if (concurrent) h->trsv_blocks = std::max(dev->sm_count, h->trsv_blocks_full / (int)dev->helpers.size());
    else h->trsv_blocks = h->trsv_blocks_full;
    // budget: the helper's k_unpack_inputs reads max_outer from the staged inputs
    double *in = HK.pin + HK.fb.out_doubles;
    in[0] = K.pin[K.fb.out_doubles + q];
    in[1] = 1.0;
    in[2] = C.max_outer;
    if (concurrent) {
      CUDA_TRY(cudaEventRecord(dev->ev_h, s));
      CUDA_TRY(cudaStreamWaitEvent(hs, dev->ev_h, 0));
    }
    // factors (both layouts), operator values, solution / rhs, the open cycle's vectors
    CUDA_TRY(gather(hs, hd.Lx, d.Lx, d.nnz_L, q));
    CUDA_TRY(gather(hs, hd.Ux, d.Ux, d.nnz_U, q));
    CUDA_TRY(gather(hs, hd.udiag, d.udiag, n, q));
    CUDA_TRY(gather(hs, hd.Lv, d.Lv, d.nnz_L, q));
    CUDA_TRY(gather(hs, hd.Uv, d.Uv, d.nnz_U, q));
    CUDA_TRY(gather(hs, hd.A_vals, d.A_vals, d.nnz_a, q));
    CUDA_TRY(gather(hs, HK.x, K.x, n, q));
    CUDA_TRY(gather(hs, HK.sr, K.sr, n, q));
    CUDA_TRY(gather(hs, HK.w, K.w, n, q));
    for (int v = 0; v < j0; ++v) {
      CUDA_TRY(gather(hs, HK.V + (size_t)v * n, K.V + (size_t)v * nbn, n, q));
      CUDA_TRY(gather(hs, HK.Z + (size_t)v * n, K.Z + (size_t)v * nbn, n, q));
    }
    h->launches += 9 + 2 * j0;
    calls[i].resume = 1;
    calls[i].T = 0;
    calls[i].b = HK.sr;
    calls[i].x0 = HK.sx0;
    calls[i].xout = HK.sx;
    Runner RH(h, calls[i]);
    k_handoff_state<<<1, 256, 0, hs>>>(R.c, RH.c, q, j0, K.beta, HK.beta);
    CUDA_TRY(cudaGetLastError());
    h->launches++;
    if ((rc = get_graph(h, RH, calls[i], graphs[i]))) return rc;
    CUDA_TRY(cudaGraphLaunch(graphs[i]->exec, hs));
    // x back into the batch's solution (interleaved column q)
    k_scatter_col<<<G, 256, 0, hs>>>(K.sx, HK.sx, n, nbp, q);
    CUDA_TRY(cudaGetLastError());
    h->launches++;
  }
  for (size_t i = 0; i < handed.size(); ++i) {
    Device *h = dev->helpers[i];
    CUDA_TRY(cudaStreamSynchronize(concurrent ? h->stream : s));
    const FgGraph *g = graphs[i];
    const int *ctrl = h->kry->pin_ctrl;
    h->launches += g->l_pro + (long long)ctrl[C.m + 2] * g->l_iter + g->l_epi;
    // cycles the helper ran (its count continued the batch's)
    h->launches += (long long)std::max(0, ctrl[C.m + 1] - (K.pin_ctrl[C.m + 1] - 1)) * g->l_cyc;
    dev->launches += h->launches;
    h->launches = 0;
  }
  return KKT_OK;
}

int dev_fgmres(Device *dev, const double *b, const double *x0, double *xout, const kkt_krylov_cfg *cfg,
               int mode, const int *active_in, const kkt_linop *opK, const kkt_linop *opM,
               kkt_krylov_report *rep, double *hist, int hist_cap, double *rpairs, int rp_cap,
               const std::function<int()> *post) {
  DevPlan &d = dev->d;
  const int nb = d.nb;
  if (cfg->m < 1) return set_error(KKT_ERR_BAD_ARG, "restart length m must be >= 1");
  if (cfg->m > 62) return set_error(KKT_ERR_BAD_ARG, "restart length m must be <= 62");
  if (cfg->max_outer < 0) return set_error(KKT_ERR_BAD_ARG, "max_outer must be >= 0");
  if (!dev->kry || dev->kry->m < cfg->m)
    return set_error(KKT_ERR_BAD_ARG, "FGMRES workspace smaller than m (ensure_krylov first)");
  const bool callbacks = op_kind(opK) == KKT_OP_CALLBACK || op_kind(opM) == KKT_OP_CALLBACK;
  if ((op_kind(opK) != KKT_OP_HANDLE || op_kind(opM) != KKT_OP_HANDLE) && d.nbp != 1)
    return set_error(KKT_ERR_BAD_ARG, "generic operators need a single-system handle");
  int rc = ensure_control(dev, cfg->m, std::max(cfg->max_outer, 1));
  if (rc) return rc;
  Krylov &K = *dev->kry;
  const FgBufs &B = K.fb;
  // stage the per-system tolerances / active flags / budget (pinned, read by the graph)
  double *in = K.pin + B.out_doubles;
  const int nbp = d.nbp;
  for (int q = 0; q < nbp; ++q) {
    const double tq = q < nb ? (mode == 1 ? (cfg->delta_sys ? cfg->delta_sys[q] : cfg->delta_tol)
                                          : (cfg->delta_sys ? cfg->delta_sys[q] : cfg->tol))
                             : 1.0;
    if (q < nb && !(tq > 0)) return set_error(KKT_ERR_BAD_ARG, mode == 1 ? "delta_tol must be positive"
                                                                      : "tol must be positive");
    in[q] = tq;
    in[nbp + q] = (q < nb && (!active_in || active_in[q])) ? 1.0 : 0.0;
  }
  in[2 * nbp] = cfg->max_outer;
  const bool host_loop = callbacks || (cfg->flags & KKT_FG_HOST_LOOP) || std::getenv("KKT_FG_HOST_LOOP");
  // A graph runs on the workspace's fixed vectors (b -> sr, x0 -> sx0, x -> sx), so one
  // captured graph serves every call whatever the caller's pointers: stage around it.
  const size_t vbytes = 8 * (size_t)nbp * d.n;
  if (!host_loop) {
    if (x0 != K.sx0) CUDA_TRY(cudaMemcpyAsync(K.sx0, x0, vbytes, cudaMemcpyDeviceToDevice, dev->stream));
    if (b != K.sr) CUDA_TRY(cudaMemcpyAsync(K.sr, b, vbytes, cudaMemcpyDeviceToDevice, dev->stream));
  }
  const int T = (!host_loop && nbp > 1 && !(cfg->flags & KKT_FG_NO_HANDOFF)) ? handoff_threshold(nb) : 0;
  Call C{host_loop ? b : K.sr, host_loop ? x0 : K.sx0, host_loop ? xout : K.sx, cfg->m, cfg->max_outer, mode,
         (cfg->flags & KKT_FG_STATS_AFTER) ? 1 : 0, (cfg->flags & KKT_FG_MGS) ? 1 : 0, opK, opM};
  C.T = T;
  Runner R(dev, C);
  std::vector<int> handed;
  if (host_loop) {
    rc = R.run_host();
    if (rc) return rc;
  } else {
    FgGraph *G = nullptr;
    if ((rc = get_graph(dev, R, C, G))) return rc;
    CUDA_TRY(cudaGraphLaunch(G->exec, dev->stream));
    // the copies of x behind the graph, then the call's one synchronisation
    if (xout != K.sx) CUDA_TRY(cudaMemcpyAsync(xout, K.sx, vbytes, cudaMemcpyDeviceToDevice, dev->stream));
    if (post && (rc = (*post)())) return rc;
    CUDA_TRY(cudaStreamSynchronize(dev->stream));
    const int *ctrl = K.pin_ctrl;
    dev->launches += G->l_pro + (long long)ctrl[cfg->m + 1] * G->l_cyc + (long long)ctrl[cfg->m + 2] * G->l_iter +
                     G->l_epi;
    if (T > 0 && ctrl[cfg->m + 6] > 0)
      for (int q = 0; q < nb; ++q)
        if (K.pin[(size_t)q * FG_REP + 19] > 0) handed.push_back(q);
  }
  // the stragglers: helpers resume them (their reports replace the batch's)
  std::vector<const double *> src(nb, nullptr);
  std::vector<int> src_hcap(nb, K.c_hcap), src_rpcap(nb, K.c_rpcap);
  if (!handed.empty()) {
    if ((rc = resume_handed(dev, R, C, handed))) return rc;
    for (size_t i = 0; i < handed.size(); ++i) {
      const Krylov &HK = *dev->helpers[i]->kry;
      src[handed[i]] = HK.pin;
      src_hcap[handed[i]] = HK.c_hcap;
      src_rpcap[handed[i]] = HK.c_rpcap;
    }
  }
  if (!handed.empty()) {  // the helpers changed x: repeat the copies
    if (xout != K.sx) CUDA_TRY(cudaMemcpyAsync(xout, K.sx, vbytes, cudaMemcpyDeviceToDevice, dev->stream));
    if (post && (rc = (*post)())) return rc;
    CUDA_TRY(cudaStreamSynchronize(dev->stream));
  } else if (host_loop && post) {
    if ((rc = (*post)())) return rc;
    CUDA_TRY(cudaStreamSynchronize(dev->stream));
  }
  // unpack the report blocks: [nbp][FG_REP] | history [nbp][hcap] | restart pairs [nbp][rpcap][2]
  int failed = 0;
  for (int q = 0; q < nb; ++q) {
    const bool hq = src[q] != nullptr;
    const double *ob = hq ? src[q] : K.pin;
    const int pb = hq ? 1 : nbp, qi = hq ? 0 : q, hcap = src_hcap[q], rpcap = src_rpcap[q];
    const double *o = ob + (size_t)qi * FG_REP;
    const double *oh = ob + (size_t)pb * FG_REP + (size_t)qi * hcap;
    const double *orp = ob + (size_t)pb * FG_REP + (size_t)pb * hcap + (size_t)qi * 2 * rpcap;
    kkt_krylov_report &r = rep[q];
    std::memset(&r, 0, sizeof r);
    r.iterations = (int)o[0];
    r.precond_applications = r.iterations;
    r.converged = (int)o[1];
    r.restarts = (int)o[2];
    r.beta0 = o[3];
    r.est_final = o[4];
    r.true_final = o[5];
    r.nonfinite = (int)o[6];
    r.triggered = (int)o[7];
    for (int i = 0; i < 5; ++i) r.stats_before[i] = o[8 + i];
    r.stats_before[5] = o[13];
    for (int i = 0; i < 5; ++i) r.stats_after[i] = o[14 + i];
    r.stats_after[5] = o[13];
    r.handed_off = hq ? 1 : 0;
    failed |= r.nonfinite;
    if (hist) {
      const int nh = std::min(std::min(r.iterations + 1, hcap), hist_cap);
      for (int i = 0; i < nh; ++i) hist[(size_t)q * hist_cap + i] = oh[i];
    }
    if (rpairs) {
      const int np = std::min(std::min(r.restarts, rpcap), rp_cap);
      for (int i = 0; i < 2 * np; ++i) rpairs[(size_t)q * 2 * rp_cap + i] = orp[i];
    }
  }
  if (failed) return set_error(KKT_ERR_NONFINITE, "operator or preconditioner produced a non-finite entry");
  return KKT_OK;
}

}  // namespace kkt
