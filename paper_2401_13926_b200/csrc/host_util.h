// Small host-side helpers shared by the orchestration translation units.
#pragma once
#include <cuda_runtime.h>

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

struct KState {
  double beta0, beta, target, floor, est, hj1;
  int j, stop, converged, pad;
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
  KState *st = nullptr;
  double *partials = nullptr;  // [nb][m+2][rb]
  double *status = nullptr;    // [nb][4] {est|beta, stop, hj1, nonfinite}
  int *mask = nullptr, *jused = nullptr;
  void *mem = nullptr;
};

// host-side building blocks (device.cu / krylov.cu); vectors are [nb][n]
int dev_solve(Device *dev, const double *b, double *x);
int dev_spmv(Device *dev, const double *x, double *y, const double *bsub, double *nrm_partials);
int dev_residual_norms(Device *dev, const double *r, const double *x, double *out6);
int alloc_krylov(Device *dev, int m);
void free_krylov(Device *dev);
// rep / hist are per system (rep[nb], hist[nb][hist_cap]); active (may be NULL) selects the
// systems to run, the others keep x = x0 untouched semantics to the caller.
int dev_fgmres(Device *dev, const double *b, const double *x0, double *xout,
               const kkt_krylov_cfg *cfg, kkt_krylov_report *rep, double *hist, int hist_cap,
               const int *active);

}  // namespace kkt
