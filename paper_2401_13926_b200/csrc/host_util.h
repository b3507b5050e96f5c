// Small host-side helpers shared by the orchestration translation units.
#pragma once
#include <cuda_runtime.h>

#include <functional>
#include <string>
#include <vector>

#include "device.h"

namespace kkt {

#define CUDA_TRY(expr)                                                                  \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      return set_error(_e == cudaErrorMemoryAllocation ? KKT_ERR_OOM : KKT_ERR_CUDA,     \
                       std::string(#expr) + ": " + cudaGetErrorString(_e));             \
  } while (0)

// count one launch and surface launch errors
#define LAUNCH(expr)                                                                    \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    dev->launches++;                                                                    \
    if (_e != cudaSuccess)                                                              \
      return set_error(KKT_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(_e)); \
  } while (0)

inline size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

template <typename T>
inline T *carve(char *&cur, size_t count) {
  T *p = reinterpret_cast<T *>(cur);
  cur += align_up(count * sizeof(T) + 1);
  return p;
}

// Per-system FGMRES control state on the device (krylov.cu), [nbp] each.
struct FgBufs {
  double *beta0 = nullptr, *bnew = nullptr, *target = nullptr, *floor_ = nullptr, *est = nullptr,
         *hj1 = nullptr;
  int *act_in = nullptr, *active = nullptr, *running = nullptr, *cycle = nullptr, *jused = nullptr,
      *iters = nullptr, *restarts = nullptr, *converged = nullptr, *failed = nullptr, *trig = nullptr,
      *handed = nullptr, *vmask = nullptr;
  int *ctrl = nullptr;                // control words (iteration / cycle conditions, counters)
  unsigned long long *hnd = nullptr;  // conditional-node handles the control kernels set
  double *out = nullptr;              // report block | history | restart pairs (one D2H)
  double *stats0 = nullptr, *stats1 = nullptr;  // residual statistics before / after
  double *in = nullptr;               // tolerances, active flags, budget (one H2D)
  size_t out_doubles = 0, in_doubles = 0;
};

// One instantiated FGMRES graph and what it was captured for.
struct FgGraph {
  const double *b = nullptr, *x0 = nullptr;
  double *xout = nullptr;
  int m = 0, mode = 0, want_after = 0, mgs = 0, resume = 0, T = 0;
  DevPlan plan{};
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  long long l_pro = 0, l_cyc = 0, l_iter = 0, l_epi = 0;  // kernels per segment (launch counter)
};

// FGMRES(m) workspace for nb systems, allocated once per handle (krylov.cu).
struct Krylov {
  int m = 0, n = 0;
  double *V = nullptr;  // [m+1][nb][n] basis
  double *Z = nullptr;  // [m][nb][n] preconditioned basis (flexible)
  double *w = nullptr, *w1 = nullptr, *r = nullptr, *x = nullptr;  // [nb][n]
  double *sr = nullptr, *sx0 = nullptr, *sx = nullptr;             // kkt_dev_step staging
  double *h1 = nullptr, *h2 = nullptr, *H = nullptr, *cs = nullptr, *sn = nullptr, *g = nullptr,
         *yv = nullptr, *nrm = nullptr, *beta = nullptr;            // per-system small state
  double *partials = nullptr;  // [nb][m+2][rb]
  void *mem = nullptr;
  // control state (sized for (m, max_outer) on first use) and its pinned host mirror
  FgBufs fb;
  void *cmem = nullptr;
  double *pin = nullptr;
  double *cb_pin = nullptr;  // host callback operator buffers (in | out)
  int *pin_ctrl = nullptr;
  size_t pin_bytes = 0;
  int c_hcap = 0, c_rpcap = 0, c_m = 0;
  std::vector<FgGraph> graphs;
};

// Standalone operator handle (kkt_op_*): only the operator part of DevPlan is populated.
struct Operator {
  int device = 0;
  cudaStream_t stream = nullptr;
  DevPlan d{};
  void *arena = nullptr;
  double *pinned = nullptr;
  long long launches = 0;
};

// host-side building blocks (device.cu / krylov.cu); vectors are [nb][n]
int dev_solve(Device *dev, const double *b, double *x);
int dev_spmv(Device *dev, const double *x, double *y, const double *bsub, double *nrm_partials);
int dev_residual_norms(Device *dev, const double *r, const double *x, double *out6);
int alloc_krylov(Device *dev, int m);
int prepare_helpers(Device *dev);  // a batched handle's straggler helpers (krylov.cu)
int ensure_krylov(Device *dev, int m);
void free_krylov(Device *dev);
// FGMRES on every system of the handle (krylov.py:117-208).  mode 0: fgmres with tol (or
// delta_sys) on the systems active_in selects (NULL = all); mode 1: refine_fgmres
// (refine.py:103-132) - the per-system trigger ||b - K x0||_2 > delta ||b||_2 is decided on the
// device, the untriggered systems return x0.  opK / opM NULL = the handle's operator values /
// LU factors.  rep[nb]; hist[nb][hist_cap] and rpairs[nb][rp_cap][2] may be NULL.  Failing
// systems (non-finite operator output) are reported per system; the call then returns
// KKT_ERR_NONFINITE after finishing the others.
// `post` (may be null) enqueues the caller's follow-up copies of xout; it runs before the one
// host synchronisation (and again after a straggler hand-off), so a kkt_dev_step waits once.
int dev_fgmres(Device *dev, const double *b, const double *x0, double *xout, const kkt_krylov_cfg *cfg,
               int mode, const int *active_in, const kkt_linop *opK, const kkt_linop *opM,
               kkt_krylov_report *rep, double *hist, int hist_cap, double *rpairs, int rp_cap,
               const std::function<int()> *post = nullptr);

}  // namespace kkt
