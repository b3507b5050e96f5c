// sm_100a kernels of the per-system hot path.  FP64 CUDA-core work (there is no dense
// contraction anywhere on this path, so tcgen05/TMEM do not apply).  All arithmetic that the
// reference performs as numpy elementwise ops is written with explicit round-to-nearest
// intrinsics and the TU is compiled with --fmad=false, so products and differences round
// separately exactly like numpy's `x - (l*xk)`.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace kkt {

constexpr int WARP = 32;

__device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int *p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ double ldcg(const double *p) { return __ldcg(p); }

// ---- value-as-flag readiness ---------------------------------------------------------
// Buffers that other warps wait on are reset to an all-ones NaN bit pattern (memset 0xFF).
// Arithmetic never produces that pattern (canonical NaNs differ) and producers canonicalize
// it away (`unsentinel`), so "value != sentinel" means "value published".  An aligned 8-byte
// store is single-copy atomic, so no separate flag or fence is needed.
constexpr unsigned long long SENTINEL_BITS = 0xFFFFFFFFFFFFFFFFull;

__device__ __forceinline__ bool is_sentinel(double v) {
  return (unsigned long long)__double_as_longlong(v) == SENTINEL_BITS;
}
__device__ __forceinline__ double unsentinel(double v) {
  return is_sentinel(v) ? __longlong_as_double(0x7FF8000000000000ll) : v;
}
__device__ __forceinline__ double ld_relaxed_f64(const double *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return __longlong_as_double((long long)v);
}
__device__ __forceinline__ void st_relaxed_f64(double *p, double v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(__double_as_longlong(v))
               : "memory");
}
// Spin (optionally backing off with __nanosleep(sleep_ns) after a few tries) until *p is
// published.
__device__ __forceinline__ double wait_value(const double *p, int sleep_ns = 0) {
  double v = ld_relaxed_f64(p);
  for (int it = 0; is_sentinel(v); ++it) {
    if (sleep_ns && it > 4) __nanosleep(sleep_ns);
    v = ld_relaxed_f64(p);
  }
  return v;
}
// Exponential back-off variant for addresses many warps may wait on at once (hot spots):
// polling pressure on one L2 slice would otherwise delay the producer's own store.
__device__ __forceinline__ double wait_value_backoff(const double *p) {
  double v = ld_relaxed_f64(p);
  unsigned ns = 16;
  while (is_sentinel(v)) {
    __nanosleep(ns);
    ns = ns < 256 ? 2 * ns : 256;
    v = ld_relaxed_f64(p);
  }
  return v;
}

// Back-off poll for batched kernels, where hundreds of warps can be waiting at once: a tight
// spin from every waiter saturates L2 and slows the very producers being waited on.
__device__ __forceinline__ double wait_value_bo(const double *p, int cap_ns) {
  double v = ld_relaxed_f64(p);
  unsigned ns = 32;
  while (is_sentinel(v)) {
    __nanosleep(ns);
    ns = ns < (unsigned)cap_ns ? 2 * ns : (unsigned)cap_ns;
    v = ld_relaxed_f64(p);
  }
  return v;
}

// ---- cp.async (LDGSTS) helpers for shared-memory prefetch rings ----------------------
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ double ld_volatile_shared(const volatile double *p) { return *p; }

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned long long dbits(double v) {
  return (unsigned long long)__double_as_longlong(v);
}

// Max / min of non-negative doubles via their (monotone) bit patterns.
__device__ __forceinline__ void atomic_max_nonneg(unsigned long long *a, double v) {
  if (v > 0.0) atomicMax(a, dbits(v));
}
__device__ __forceinline__ void atomic_min_nonneg(unsigned long long *a, double v) {
  atomicMin(a, dbits(v));
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Fixed-shape (deterministic) block sum of `v` across blockDim.x threads.
template <int BLOCK>
__device__ __forceinline__ double block_sum(double v, double *sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = (l < BLOCK / 32) ? sh[l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
  }
  return r;  // valid in thread 0
}

}  // namespace kkt
