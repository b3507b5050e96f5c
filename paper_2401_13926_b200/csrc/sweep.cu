// Blocked sweep over the dense trailing block of the triangular solves (direct_lu.py:359-379),
// for the single-system and the batched interleaved handles (S systems per CTA).
//
// The reference sweeps columns one at a time; every row accumulates its updates in column
// order (ascending for L, descending for U) with separately rounded products.  Here the
// block's columns are taken 32 at a time:
//   phase A (one warp per system): the 32x32 diagonal triangle as a register chain — lane i
//     owns row lo+i; at step t lane t's value is final (y_t; for U after the division by
//     u_tt) and is broadcast with one shuffle, and every lane holding L(i,t) / U(i,t)
//     subtracts its product.  The triangle's values were prefetched into shared memory with
//     cp.async while the previous block ran.
//   phase B (all threads): every later row with entries in the block's columns applies them
//     in its CSR order from the block's y values in shared memory.
// Per row the subtractions therefore happen in exactly the reference's order (bitwise), but
// the sweep costs one shuffle chain step per column and two CTA barriers per 32 columns,
// instead of one barrier per column.
#include <cuda_runtime.h>

#include <cstdlib>

#include "device.h"
#include "kernels.cuh"

namespace kkt {

// threads per sweep CTA (template NT; KKT_SWEEP_THREADS = 256 | 512 | 1024): phase A is one
// warp per system whatever NT; the other warps stage the next block and run phase B.
// MODE 0: off-diagonal runs read from global in phase B; 1: staged into shared memory by the
// non-chain warps while the chain runs; 2 (look-ahead): block c+1's tile AND runs are staged
// (double-buffered) while block c's chain runs, so a block's critical path is barrier ->
// chain -> barrier -> phase B from shared memory, with no load latency on it.
template <bool IS_U, int S, int MODE, int NT>
__global__ void __launch_bounds__(NT) k_trsv_blocked(DevPlan d, double *__restrict__ xout) {
  constexpr int BS_THREADS = NT;
  constexpr bool STAGED = MODE >= 1;
  extern __shared__ double sm[];
  const SweepDev &sw = IS_U ? d.swU : d.swL;
  const int sys0 = blockIdx.x * S;
  bool any = false;
#pragma unroll
  for (int q = 0; q < S; ++q) any |= sys_active(d, sys0 + q);
  if (!any) return;  // uniform over the CTA (inactive systems of an active CTA are harmless:
                     // they replay their previous solve's tail from their own state)
  const int p = IS_U ? d.pU : d.pL;
  const int T = d.n - p;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double *acc = sm;                          // [T][S]
  double *tile = acc + (size_t)T * S;        // [2][32*32][S]
  double *yb = tile + 2 * 1024 * S;          // [32][S]
  constexpr int NBUF = MODE == 2 ? 2 : 1;
  double *sv = yb + 32 * S;                  // [NBUF][max_stage][S]   (STAGED)
  int *scol = reinterpret_cast<int *>(sv + (size_t)NBUF * sw.max_stage * S);  // [NBUF][max_stage]
  const double *vals = IS_U ? d.Uv : d.Lv;
  const int *ci = IS_U ? d.Uci : d.Lci;
  for (int f = tid; f < T * S; f += BS_THREADS) {
    const int r = p + f / S, q = f % S, sys = sys0 + q;
    if (IS_U) {
      acc[f] = ldcg(&d.yL[IL(d, r, sys)]);  // L result of the head rows
      d.yL[IL(d, r, sys)] = __longlong_as_double((long long)SENTINEL_BITS);  // next solve
    } else {
      acc[f] = ldcg(&d.tacc[IL(d, r - p, sys)]);  // b_perm - sum over columns < p (grid phase)
      d.yU[IL(d, r, sys)] = __longlong_as_double((long long)SENTINEL_BITS);
    }
  }
  auto issue_tile = [&](int c, int t0, int nthr) {
    if (c < sw.nblk) {
      double *tl = tile + (size_t)(c & 1) * 1024 * S;
      const int k0 = sw.dptr[c], k1 = sw.dptr[c + 1];
      for (int f = t0; f < (k1 - k0) * S; f += nthr) {
        const int k = k0 + f / S, q = f % S;
        cp_async8(&tl[(size_t)sw.ddst[k] * S + q], &vals[IL(d, sw.dsrc[k], sys0 + q)]);
      }
    }
    cp_async_commit();
  };
  // MODE 2: block c's off-diagonal runs into stage buffer c & 1 (issued a block ahead)
  auto issue_runs = [&](int c, int t0, int nthr) {
    if (c < sw.nblk) {
      double *svb = sv + (size_t)(c & 1) * sw.max_stage * S;
      int *scb = scol + (size_t)(c & 1) * sw.max_stage;
      const int b0 = sw.bptr[c], b1 = sw.bptr[c + 1];
      for (int k = b0 + t0; k < b1; k += nthr) {
        const int beg = sw.bbeg[k], cnt = sw.bcnt[k], o = sw.bofs[k];
        for (int e = 0; e < cnt; ++e) {
#pragma unroll
          for (int q = 0; q < S; ++q) cp_async8(&svb[(size_t)(o + e) * S + q], &vals[IL(d, beg + e, sys0 + q)]);
          cp_async4(&scb[o + e], &ci[beg + e]);
        }
      }
    }
  };
  if (MODE == 2) issue_runs(0, tid, BS_THREADS);
  issue_tile(0, tid, BS_THREADS);  // (commits the group: tile 0 + the runs of block 0)
  bool bad = false;
  // optional timeline (KKT_TRACE, single system): per block {top, tiles ready, y ready, end}
  unsigned long long *tr = (d.trace_trsv && blockIdx.x == 0 && tid == 0)
                               ? d.trace_trsv + (IS_U ? (size_t)d.n : 0) + p : nullptr;
#pragma unroll 1
  for (int c = 0; c < sw.nblk; ++c) {
    if (tr) tr[4 * c] = globaltimer();
    int lo, w;
    if (!IS_U) {
      lo = p + 32 * c;
      w = min(32, d.n - lo);
    } else {
      const int hi = d.n - 32 * c;
      lo = max(p, hi - 32);
      w = hi - lo;
    }
    // per-lane inputs of phase A, loaded before the barrier (independent of the chain)
    const int s = warp;
    const bool chain = warp < S;
    unsigned mask = 0;
    double piv = 1.0;
    if (chain && lane < w) {
      mask = sw.dmask[c * 32 + lane];
      if (IS_U) piv = d.udiag[IL(d, lo + lane, sys0 + s)];
    }
    if (MODE == 2) {
      cp_async_wait<0>();  // this thread's copies of block c (tile + runs) have landed
    } else {
      issue_tile(c + 1, tid, BS_THREADS);
      cp_async_wait<1>();  // this thread's copies of tile c have landed
    }
    __syncwarp();        // (the copy loops leave warps diverged; the barrier is .aligned)
    __syncthreads();     // ... everyone's; and phase B of block c-1 is complete
    if (tr) tr[4 * c + 1] = globaltimer();
    const int b0 = sw.bptr[c], b1 = sw.bptr[c + 1];
    if (MODE == 2 && warp >= S) {  // the other warps stage block c+1 while the chain runs
      issue_runs(c + 1, tid - 32 * S, BS_THREADS - 32 * S);
      issue_tile(c + 1, tid - 32 * S, BS_THREADS - 32 * S);
    }
    if (MODE == 1 && warp >= S) {  // the other warps stream the block's off-diagonal runs
      for (int k = b0 + tid - 32 * S; k < b1; k += BS_THREADS - 32 * S) {
        const int beg = sw.bbeg[k], cnt = sw.bcnt[k], o = sw.bofs[k];
        for (int e = 0; e < cnt; ++e) {
#pragma unroll
          for (int q = 0; q < S; ++q) cp_async8(&sv[(size_t)(o + e) * S + q], &vals[IL(d, beg + e, sys0 + q)]);
          cp_async4(&scol[o + e], &ci[beg + e]);
        }
      }
    }
    if (MODE == 1) cp_async_commit();
    if (chain) {
      // the lane's row of the diagonal triangle in registers, then a pure register chain
      const double *tl = tile + (size_t)(c & 1) * 1024 * S;
      double lrow[32];
#pragma unroll
      for (int t = 0; t < 32; ++t) lrow[t] = ((mask >> t) & 1u) ? tl[(size_t)(lane * 32 + t) * S + s] : 0.0;
      double a = lane < w ? acc[(size_t)(lo + lane - p) * S + s] : 0.0;
      double y = 0.0;
      if (!IS_U) {
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          if (t >= w) break;
          const double yt = __shfl_sync(0xffffffffu, a, t);  // row lo+t is final
          if ((mask >> t) & 1u) a = __dsub_rn(a, __dmul_rn(lrow[t], yt));
        }
        y = a;
      } else {
#pragma unroll
        for (int t = 31; t >= 0; --t) {
          if (t >= w) continue;
          double yl = 0.0;
          if (lane == t) yl = __ddiv_rn(a, piv);  // y_t = acc_t / u_tt
          const double yt = __shfl_sync(0xffffffffu, yl, t);
          if (lane == t) y = yt;
          if ((mask >> t) & 1u) a = __dsub_rn(a, __dmul_rn(lrow[t], yt));
        }
      }
      if (tr) tr[4 * c + 2] = globaltimer();
      if (lane < w) {
        const int j = lo + lane, sys = sys0 + s;
        yb[lane * S + s] = y;
        if (IS_U) {
          st_relaxed_f64(&d.yU[IL(d, j, sys)], unsentinel(y));
          xout[IL(d, d.col_perm[j], sys)] = y;
          if (!isfinite(y)) bad = true;
        } else {
          st_relaxed_f64(&d.yL[IL(d, j, sys)], unsentinel(y));
        }
      }
    }
    if (MODE == 1) cp_async_wait<0>();
    __syncwarp();
    __syncthreads();  // the block's y values (and staged runs) are in shared memory
    // phase B: later rows (L: below the block; U: above it, inside the head) in CSR order
    if (STAGED) {
      const double *svb = sv + (size_t)(MODE == 2 ? (c & 1) : 0) * sw.max_stage * S;
      const int *scb = scol + (size_t)(MODE == 2 ? (c & 1) : 0) * sw.max_stage;
      for (int f = tid; f < (b1 - b0) * S; f += BS_THREADS) {
        const int k = b0 + f / S, q = f % S;
        const int r = sw.brow[k], cnt = sw.bcnt[k], o = sw.bofs[k];
        double a = acc[(size_t)(r - p) * S + q];
#pragma unroll 4
        for (int e = 0; e < cnt; ++e)
          a = __dsub_rn(a, __dmul_rn(svb[(size_t)(o + e) * S + q], yb[(scb[o + e] - lo) * S + q]));
        acc[(size_t)(r - p) * S + q] = a;
      }
      if (tr) tr[4 * c + 3] = globaltimer();
      continue;
    }
    for (int f = tid; f < (b1 - b0) * S; f += BS_THREADS) {
      const int k = b0 + f / S, q = f % S, sys = sys0 + q;
      const int r = sw.brow[k], beg = sw.bbeg[k], cnt = sw.bcnt[k];
      double a = acc[(size_t)(r - p) * S + q];
      for (int e0 = 0; e0 < cnt; e0 += 8) {
        int cl[8];
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (e0 + u < cnt) {
            cl[u] = ci[beg + e0 + u];
            v[u] = vals[IL(d, beg + e0 + u, sys)];
          }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (e0 + u < cnt) a = __dsub_rn(a, __dmul_rn(v[u], yb[(cl[u] - lo) * S + q]));
      }
      acc[(size_t)(r - p) * S + q] = a;
    }
  }
  cp_async_wait<0>();
  if (IS_U && bad) atomicOr(&d.scal[(size_t)(sys0 + warp) * SCAL_STRIDE + SC_NONFINITE], 1ull);
}

constexpr size_t SMEM_CAP = 227 * 1024;
constexpr int SWEEP_THREADS_DEFAULT = 256;

static size_t blocked_smem(int T, int S, int stage, int nbuf = 1) {
  return ((size_t)T * S + 2 * 1024 * S + 32 * S + (size_t)nbuf * stage * S) * sizeof(double) +
         (size_t)nbuf * stage * sizeof(int);
}

template <bool IS_U, int S, int MODE, int NT>
static cudaError_t set_attr() {
  return cudaFuncSetAttribute(k_trsv_blocked<IS_U, S, MODE, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)SMEM_CAP);
}

template <int S, int NT>
static cudaError_t set_attrs() {
  cudaError_t e = set_attr<false, S, 0, NT>();
  if (e == cudaSuccess) e = set_attr<true, S, 0, NT>();
  if (e == cudaSuccess) e = set_attr<false, S, 1, NT>();
  if (e == cudaSuccess) e = set_attr<true, S, 1, NT>();
  if (e == cudaSuccess) e = set_attr<false, S, 2, NT>();
  if (e == cudaSuccess) e = set_attr<true, S, 2, NT>();
  return e;
}

static int sweep_threads() {
  const char *e = std::getenv("KKT_SWEEP_THREADS");
  const int t = e ? std::atoi(e) : SWEEP_THREADS_DEFAULT;
  return t >= 1024 ? 1024 : t >= 512 ? 512 : 256;
}

cudaError_t sweep_configure() {
  cudaError_t e = set_attrs<1, 256>();
  if (e == cudaSuccess) e = set_attrs<2, 256>();
  if (e == cudaSuccess) e = set_attrs<4, 256>();
  if (e == cudaSuccess) e = set_attrs<1, 512>();
  if (e == cudaSuccess) e = set_attrs<1, 1024>();
  return e;
}

template <bool IS_U, int S, int MODE>
static void launch_nt(const DevPlan &d, double *x, size_t smem, cudaStream_t s) {
  const int nt = S == 1 ? sweep_threads() : 256;
  if (nt == 1024) k_trsv_blocked<IS_U, S, MODE, 1024><<<d.nbp / S, 1024, smem, s>>>(d, x);
  else if (nt == 512) k_trsv_blocked<IS_U, S, MODE, 512><<<d.nbp / S, 512, smem, s>>>(d, x);
  else k_trsv_blocked<IS_U, S, MODE, 256><<<d.nbp / S, 256, smem, s>>>(d, x);
}

template <bool IS_U, int S>
static void launch_mode(const DevPlan &d, double *x, int mode, size_t smem, cudaStream_t s) {
  if (mode == 2) launch_nt<IS_U, S, 2>(d, x, smem, s);
  else if (mode == 1) launch_nt<IS_U, S, 1>(d, x, smem, s);
  else launch_nt<IS_U, S, 0>(d, x, smem, s);
}

// the staged variant when a block's runs fit in shared memory, else runs from global.  The
// look-ahead variant (KKT_SWEEP_AHEAD=1, two blocks' runs in shared memory) is bitwise too but
// measured slower (10k: batch pair 1.85 -> 2.02 ms, single 1.24 -> 1.28 ms): the blocks are
// bound by their chains and barriers, not by the staging latency it hides.
template <int S>
static void launch_s(const DevPlan &d, bool upper, double *x, int T, cudaStream_t s) {
  const SweepDev &sw = upper ? d.swU : d.swL;
  const char *na = std::getenv("KKT_SWEEP_AHEAD");
  const bool ahead = na && std::atoi(na) != 0;
  const bool no_stage = std::getenv("KKT_SWEEP_NOSTAGE") != nullptr;
  const size_t s2 = blocked_smem(T, S, sw.max_stage, 2), s1 = blocked_smem(T, S, sw.max_stage, 1);
  int mode = 0;
  size_t smem = blocked_smem(T, S, 0);
  if (!no_stage && ahead && s2 <= SMEM_CAP) mode = 2, smem = s2;
  else if (!no_stage && s1 <= SMEM_CAP) mode = 1, smem = s1;
  if (upper) launch_mode<true, S>(d, x, mode, smem, s);
  else launch_mode<false, S>(d, x, mode, smem, s);
}

cudaError_t launch_sweep_blocked(const DevPlan &d, bool upper, double *x, cudaStream_t s) {
  const int T = d.n - (upper ? d.pU : d.pL);
  if (T <= 0) return cudaSuccess;
  // systems per CTA: one CTA per system spreads a batch over the SMs (the sweep is a chain
  // of short steps, so parallel CTAs beat coalescing); KKT_SWEEP_S=2|4 packs more
  static const int SB = std::getenv("KKT_SWEEP_S") ? std::atoi(std::getenv("KKT_SWEEP_S")) : 1;
  if (d.nbp == 1 || SB <= 1) launch_s<1>(d, upper, x, T, s);
  else if (SB == 2) launch_s<2>(d, upper, x, T, s);
  else launch_s<4>(d, upper, x, T, s);
  return cudaGetLastError();
}

}  // namespace kkt
