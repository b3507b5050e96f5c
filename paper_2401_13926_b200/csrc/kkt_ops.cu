// KKT value assembly, right-hand-side reduction and bound-multiplier recovery on the device
// (kkt.assemble_kkt / assemble_rhs / recover_dz, kkt.py:88-144): the
// steps either side of the solve in an interior-point iteration, so a batched IPM ships
// only H, J, x, z and mu per system instead of assembled matrices.  Elementwise work,
// HBM-bound; arithmetic and grouping exactly as numpy's (bitwise equal K values / rhs / dz).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../../include/kktb200.h"
#include "kkt_internal.h"

namespace kkt {

// K values [nb][nnz_K]: position p sums its sources in the reference's np.add.at order
// (H entries, then D_x = z / x, then J entries; kkt.py:104-107).  src[p][0..1]: ids into
// [H | D | J] (-1: none); 0 + a == a exactly, so the first source is taken as is.
__global__ void k_assemble_values(int64_t nnz_K, int64_t n, int64_t nH, int64_t nJ, int nb,
                                  const int2 *__restrict__ src, const double *__restrict__ H,
                                  const double *__restrict__ J, const double *__restrict__ x,
                                  const double *__restrict__ z, double *__restrict__ K) {
  const int64_t total = nnz_K * nb;
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < total;
       f += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(f / nnz_K);
    const int64_t p = f - (int64_t)s * nnz_K;
    const int2 sp = src[p];
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int id = q == 0 ? sp.x : sp.y;
      if (id < 0) continue;
      double a;
      if (id < nH) a = H[(size_t)s * nH + id];
      else if (id < nH + n) a = __ddiv_rn(z[(size_t)s * n + (id - nH)], x[(size_t)s * n + (id - nH)]);
      else a = J[(size_t)s * nJ + (id - nH - n)];
      v = q == 0 ? a : __dadd_rn(v, a);
    }
    K[f] = v;
  }
}

// rhs [nb][n+m] = [r~_x + (z - mu / x); r_lambda]   (kkt.py:136, the reference's grouping)
__global__ void k_assemble_rhs(int64_t n, int64_t m, int nb, const double *__restrict__ rtx,
                               const double *__restrict__ rl, const double *__restrict__ x,
                               const double *__restrict__ z, const double *__restrict__ mu,
                               double *__restrict__ rhs) {
  const int64_t w = n + m, total = w * nb;
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < total;
       f += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(f / w);
    const int64_t i = f - (int64_t)s * w;
    if (i < n) {
      const size_t k = (size_t)s * n + i;
      rhs[f] = __dadd_rn(rtx[k], __dsub_rn(z[k], __ddiv_rn(mu[s], x[k])));
    } else {
      rhs[f] = rl[(size_t)s * m + (i - n)];
    }
  }
}

// dz [nb][n] = (r_z - z * dx) / x   (kkt.py:144); dx of system s at dx + s * dx_stride
__global__ void k_recover_dz(int64_t n, int nb, int64_t dx_stride, const double *__restrict__ rz,
                             const double *__restrict__ z, const double *__restrict__ dx,
                             const double *__restrict__ x, double *__restrict__ dz) {
  const int64_t total = n * nb;
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < total;
       f += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(f / n);
    const int64_t i = f - (int64_t)s * n;
    dz[f] = __ddiv_rn(__dsub_rn(rz[f], __dmul_rn(z[f], dx[(size_t)s * dx_stride + i])), x[f]);
  }
}

static unsigned grid_for(int64_t total) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 16 * 148));
}

}  // namespace kkt

extern "C" {

int kkt_assemble_values(int64_t nnz_K, int64_t n, int64_t nH, int64_t nJ, int nb,
                        const int32_t *src_dev, const double *H_dev, const double *J_dev,
                        const double *x_dev, const double *z_dev, double *K_dev, void *stream) {
  if (!src_dev || !K_dev || nb < 1 || nnz_K < 0 || n < 0 || nH < 0 || nJ < 0)
    return kkt::set_error(KKT_ERR_BAD_ARG, "kkt_assemble_values: bad argument");
  if (nnz_K == 0) return KKT_OK;
  kkt::k_assemble_values<<<kkt::grid_for(nnz_K * nb), 256, 0, (cudaStream_t)stream>>>(
      nnz_K, n, nH, nJ, nb, reinterpret_cast<const int2 *>(src_dev), H_dev, J_dev, x_dev, z_dev, K_dev);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? KKT_OK : kkt::set_error(KKT_ERR_CUDA, cudaGetErrorString(e));
}

int kkt_assemble_rhs(int64_t n, int64_t m, int nb, const double *r_tilde_x, const double *r_lambda,
                     const double *x, const double *z, const double *mu_dev, double *rhs, void *stream) {
  if (!rhs || nb < 1 || n < 0 || m < 0) return kkt::set_error(KKT_ERR_BAD_ARG, "kkt_assemble_rhs: bad argument");
  if (n + m == 0) return KKT_OK;
  kkt::k_assemble_rhs<<<kkt::grid_for((n + m) * nb), 256, 0, (cudaStream_t)stream>>>(
      n, m, nb, r_tilde_x, r_lambda, x, z, mu_dev, rhs);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? KKT_OK : kkt::set_error(KKT_ERR_CUDA, cudaGetErrorString(e));
}

int kkt_recover_dz(int64_t n, int nb, int64_t dx_stride, const double *r_z, const double *z,
                   const double *dx, const double *x, double *dz, void *stream) {
  if (!dz || nb < 1 || n < 0) return kkt::set_error(KKT_ERR_BAD_ARG, "kkt_recover_dz: bad argument");
  if (n == 0) return KKT_OK;
  kkt::k_recover_dz<<<kkt::grid_for(n * nb), 256, 0, (cudaStream_t)stream>>>(n, nb, dx_stride, r_z, z,
                                                                             dx, x, dz);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? KKT_OK : kkt::set_error(KKT_ERR_CUDA, cudaGetErrorString(e));
}

}  // extern "C"
