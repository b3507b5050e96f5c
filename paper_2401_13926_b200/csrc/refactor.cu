// Numeric refactorization on the frozen schedule (direct_lu.refactorize, direct_lu.py:297-356).
//
// Persistent warp-per-column kernel, sync-free.  Columns are dispatched in DAG-level order
// through an atomic ticket.  Column j's workspace x (its pattern: U rows, diagonal, L rows
// — sorted positions) lives in shared memory.  The warp replays so(j) in the reference's
// topological order; each update pair carries its precomputed workspace slot.
//
// Readiness without flags: every L entry is reset to a sentinel NaN bit pattern before the
// launch, and a consumer simply re-reads an entry of L(:,k) until it is no longer the
// sentinel — the producer's store of the value is the signal (no fences, one L2 round trip
// per dependency hop).  Update pairs are staged in shared memory a chunk at a time so the
// L2 latency overlaps across up to REFACTOR_STAGE pairs; the sequential replay then runs
// from shared memory.  Products and differences are rounded separately (no FMA) and every
// workspace entry receives its updates in the reference order => bitwise equal factors.
#include <cuda_runtime.h>

#include "device.h"
#include "kernels.cuh"

namespace kkt {

// ----------------------------------------------------------------------------
// Operator values: expand caller layout -> general CSR, inf-norms, max|a|.
// One thread per row; sums in entry order (np.bincount order => bitwise).
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_expand_norms(DevPlan d) {
  __shared__ double sh[3][8];
  double mx = 0.0, sg = 0.0, op = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d.n; i += gridDim.x * blockDim.x) {
    const int b = d.A_rp[i], s = d.A_split[i], e = d.A_rp[i + 1];
    double g = 0.0, s1 = 0.0, s2 = 0.0;
    for (int p = b; p < e; ++p) {
      const double v = d.in_vals[d.sym_lower ? d.gen_src[p] : p];
      d.A_vals[p] = v;
      const double a = fabs(v);
      g = __dadd_rn(g, a);
      if (p < s) s1 = __dadd_rn(s1, a); else s2 = __dadd_rn(s2, a);
      mx = fmax(mx, a);
    }
    // refactorize uses inf_norm of the general matrix (direct_lu.py:318); nsr/nrbe use the
    // operator's: two bincounts for symmetric-lower storage (sparsecore.py:339-342).
    sg = fmax(sg, g);
    op = fmax(op, d.sym_lower ? __dadd_rn(s1, s2) : g);
  }
  // maxima are order-independent: warp + block max, then one atomic per block
  mx = warp_max(mx);
  sg = warp_max(sg);
  op = warp_max(op);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sh[0][w] = mx;
    sh[1][w] = sg;
    sh[2][w] = op;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double m = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) m = fmax(m, sh[threadIdx.x][q]);
    const int slot = threadIdx.x == 0 ? SC_MAXABS_A : threadIdx.x == 1 ? SC_INFNORM : SC_OPNORM;
    atomic_max_nonneg(&d.scal[slot], m);
  }
}

__global__ void __launch_bounds__(256) k_refactor(DevPlan d) {
  // eps_patch = 1e-12 * inf_norm(Ag)                                       (:318)
  const double eps =
      __dmul_rn(PATCH_RELATIVE_FLOOR, __longlong_as_double((long long)d.scal[SC_INFNORM]));
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int wstride = d.maxpat + REFACTOR_STAGE + REFACTOR_STAGE / 2;  // doubles per warp
  double *x = smem + (size_t)wib * wstride;
  double *st_l = x + d.maxpat;
  int *st_s = reinterpret_cast<int *>(st_l + REFACTOR_STAGE);
  while (true) {
    int idx = 0;
    if (lane == 0) idx = d.ref_start + atomicAdd(d.ticket, 1);
    idx = __shfl_sync(0xffffffffu, idx, 0);
    if (idx >= d.n) break;
    const int j = d.col_order[idx];
    if (d.trace_ref && lane == 0) d.trace_ref[2 * j] = globaltimer();
    const int ub = d.Up[j], nu = d.Up[j + 1] - ub;
    const int lb = d.Lp[j], nl = d.Lp[j + 1] - lb;
    const int np = nu + 1 + nl;
    for (int s = lane; s < np; s += 32) x[s] = 0.0;
    __syncwarp();
    // x[a_tgt] = avals[a_src]                                               (:323)
    for (int q = d.ap_ptr[j] + lane; q < d.ap_ptr[j + 1]; q += 32)
      x[d.a_slot[q]] = d.A_vals[d.a_src[q]];
    __syncwarp();
    // for k in so(j) (topological): x[Li(k)] -= Lx(k) * x[k]                (:324-326)
    const int t_end = d.so_ptr[j + 1];
    int t0 = d.so_ptr[j];
    while (t0 < t_end) {
      const int t = t0 + lane;
      int4 m = make_int4(0, 0, 0, 0);
      if (t < t_end) m = d.so_meta[t];
      // inclusive scan of the pair counts => chunk of steps whose pairs fit the stage
      int incl = m.y;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const unsigned fits = __ballot_sync(0xffffffffu, t < t_end && incl <= REFACTOR_STAGE);
      int nsteps = __popc(fits);
      const bool big = nsteps == 0;  // a single step with more pairs than the stage
      if (big) nsteps = 1;
      const int pair0 = __shfl_sync(0xffffffffu, m.z, 0);
      const int npairs = big ? 0 : __shfl_sync(0xffffffffu, incl, nsteps - 1);
      // stage: 4 independent gathers per lane in flight before the shared stores
      for (int p0 = 0; p0 < npairs; p0 += 128) {
        double lv[4];
        int sv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int p = p0 + q * 32 + lane;
          if (p < npairs) {
            lv[q] = ld_relaxed_f64(&d.Lx[d.upd_lidx[pair0 + p]]);
            sv[q] = d.upd_slot[pair0 + p];
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int p = p0 + q * 32 + lane;
          if (p < npairs) {
            st_l[p] = lv[q];
            st_s[p] = sv[q];
          }
        }
      }
      __syncwarp();
      for (int i = 0; i < nsteps; ++i) {
        const int kslot = __shfl_sync(0xffffffffu, m.x, i);
        const int cnt = __shfl_sync(0xffffffffu, m.y, i);
        const int off = __shfl_sync(0xffffffffu, incl - m.y, i);
        const double xk = x[kslot];
        const int lbk = __shfl_sync(0xffffffffu, m.w, i);  // L(:,k) = Lx[lbk, lbk+cnt)
        if (!big) {
          // L(:,k) not yet published when staged?  One lane waits (with back-off) so a
          // column many warps depend on is not polled by every lane of every consumer;
          // then the whole step is re-staged with one parallel round trip.
          bool miss = false;
          for (int e = lane; e < cnt; e += 32) miss |= is_sentinel(st_l[off + e]);
          const unsigned mm = __ballot_sync(0xffffffffu, miss);
          if (mm) {
            if (lane == __ffs(mm) - 1) wait_value(&d.Lx[lbk + cnt - 1], d.poll_ns);
            __syncwarp();
            double lv[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (lane + 32 * q < cnt) lv[q] = ld_relaxed_f64(&d.Lx[lbk + lane + 32 * q]);
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (lane + 32 * q < cnt) st_l[off + lane + 32 * q] = lv[q];
            for (int e = lane + 256; e < cnt; e += 32) st_l[off + e] = ld_relaxed_f64(&d.Lx[lbk + e]);
          }
          for (int e = lane; e < cnt; e += 32) {
            double l = st_l[off + e];
            if (is_sentinel(l)) l = wait_value(&d.Lx[lbk + e]);  // rare: store not yet visible
            const int s = st_s[off + e];
            x[s] = __dsub_rn(x[s], __dmul_rn(l, xk));
          }
          if (d.trace_step && lane == 0) d.trace_step[t0 + i] = globaltimer() | (mm ? 1ull : 0ull);
        } else {
          for (int e = lane; e < cnt; e += 32) {
            const double l = wait_value_backoff(&d.Lx[lbk + e]);
            const int s = d.upd_slot[pair0 + e];
            x[s] = __dsub_rn(x[s], __dmul_rn(l, xk));
          }
        }
        __syncwarp();
      }
      t0 += nsteps;
    }
    // u_jj = x[j]; patch; L(:,j) = x[Li] / u_jj; U(:,j) = x[Ui]               (:327-344)
    // L(:,j) is what other columns wait for: publish it first, bookkeeping after.
    double gm = 0.0;
    double ujj = x[nu];
    gm = fmax(gm, fabs(ujj));
    if (fabs(ujj) < eps) {
      ujj = (ujj >= 0.0) ? eps : -eps;
      if (lane == 0) atomicAdd(&d.scal[SC_PATCHED], 1ull);
    }
    for (int s = lane; s < nl; s += 32) {
      const double v = x[nu + 1 + s];
      gm = fmax(gm, fabs(v));
      st_relaxed_f64(&d.Lx[lb + s], unsentinel(__ddiv_rn(v, ujj)));  // value == readiness
    }
    // CSR copies for the solves (scatter through the maps: batch the map loads)
    for (int s0 = 0; s0 < nl; s0 += 128) {
      int mp[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int s = s0 + 32 * q + lane;
        mp[q] = s < nl ? d.Lmap[lb + s] : 0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int s = s0 + 32 * q + lane;
        if (s < nl) d.Lv[mp[q]] = unsentinel(__ddiv_rn(x[nu + 1 + s], ujj));
      }
    }
    for (int s0 = 0; s0 < nu; s0 += 128) {
      int mp[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int s = s0 + 32 * q + lane;
        mp[q] = s < nu ? d.Umap[ub + s] : 0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int s = s0 + 32 * q + lane;
        if (s < nu) {
          const double v = x[s];
          d.Ux[ub + s] = v;
          d.Uv[mp[q]] = v;
          gm = fmax(gm, fabs(v));
        }
      }
    }
    gm = warp_max(gm);
    if (lane == 0) {
      d.udiag[j] = ujj;
      atomic_max_nonneg(&d.scal[SC_GMAX], gm);
      if (d.trace_ref) d.trace_ref[2 * j + 1] = globaltimer();
    }
    __syncwarp();
  }
}

// ----------------------------------------------------------------------------
// Wide leading levels (level 0: no replay steps; level 1: <= a few) hold most columns but
// almost no work: one thread per column, one launch per level (the kernel boundary is the
// dependency), workspace in local memory.  Same arithmetic order as k_refactor.
// ----------------------------------------------------------------------------
constexpr int SMALL_PAT = 64;

__global__ void __launch_bounds__(256) k_refactor_small(DevPlan d, int begin, int end) {
  const double eps =
      __dmul_rn(PATCH_RELATIVE_FLOOR, __longlong_as_double((long long)d.scal[SC_INFNORM]));
  const int idx = begin + blockIdx.x * blockDim.x + threadIdx.x;
  double gm = 0.0;
  if (idx < end) {
    const int j = d.col_order[idx];
    const int ub = d.Up[j], nu = d.Up[j + 1] - ub;
    const int lb = d.Lp[j], nl = d.Lp[j + 1] - lb;
    double x[SMALL_PAT];
#pragma unroll 1
    for (int s = 0; s < nu + 1 + nl; ++s) x[s] = 0.0;
    for (int q = d.ap_ptr[j]; q < d.ap_ptr[j + 1]; ++q) x[d.a_slot[q]] = d.A_vals[d.a_src[q]];
    for (int t = d.so_ptr[j]; t < d.so_ptr[j + 1]; ++t) {
      const int4 m = d.so_meta[t];
      const double xk = x[m.x];
      for (int e = 0; e < m.y; ++e) {
        const int s = d.upd_slot[m.z + e];
        x[s] = __dsub_rn(x[s], __dmul_rn(ldcg(&d.Lx[m.w + e]), xk));
      }
    }
    for (int s = 0; s < nu; ++s) {
      d.Ux[ub + s] = x[s];
      d.Uv[d.Umap[ub + s]] = x[s];
      gm = fmax(gm, fabs(x[s]));
    }
    double ujj = x[nu];
    gm = fmax(gm, fabs(ujj));
    if (fabs(ujj) < eps) {
      ujj = (ujj >= 0.0) ? eps : -eps;
      atomicAdd(&d.scal[SC_PATCHED], 1ull);
    }
    for (int s = 0; s < nl; ++s) {
      const double v = x[nu + 1 + s];
      gm = fmax(gm, fabs(v));
      const double l = unsentinel(__ddiv_rn(v, ujj));
      d.Lv[d.Lmap[lb + s]] = l;
      d.Lx[lb + s] = l;
    }
    d.udiag[j] = ujj;
    if (d.trace_ref) d.trace_ref[2 * j] = d.trace_ref[2 * j + 1] = globaltimer();
  }
  gm = warp_max(gm);
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(&d.scal[SC_GMAX], gm);
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

// ----------------------------------------------------------------------------
cudaError_t launch_expand_norms(const DevPlan &d, cudaStream_t s) {
  if (d.n) k_expand_norms<<<min((d.n + 255) / 256, 2 * 148), 256, 0, s>>>(d);
  return cudaGetLastError();
}

size_t refactor_smem_bytes(int warps, int maxpat) {
  return (size_t)warps * (maxpat + REFACTOR_STAGE + REFACTOR_STAGE / 2) * sizeof(double);
}

cudaError_t refactor_configure(int warps, size_t smem, int *blocks_per_sm) {
  cudaError_t e = cudaFuncSetAttribute(k_refactor, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(smem > 48 * 1024 ? smem : 48 * 1024));
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_refactor, 32 * warps, smem);
}

cudaError_t launch_refactor(const DevPlan &d, int blocks, int warps, size_t smem, cudaStream_t s,
                            long long *launches) {
  if (!d.n) return cudaSuccess;
  // readiness protocol: L(:,k) entries start as the sentinel
  cudaError_t e = cudaMemsetAsync(d.Lx, 0xFF, 8 * (size_t)d.nnz_L, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(d.ticket, 0, 4, s);
  if (e != cudaSuccess) return e;
  // wide leading levels: thread per column, level-synchronous
  for (int l = 0; l < d.n_small_levels; ++l) {
    const int b = d.lev_ptr[l], en = d.lev_ptr[l + 1];
    if (en > b) {
      k_refactor_small<<<(en - b + 255) / 256, 256, 0, s>>>(d, b, en);
      ++*launches;
    }
  }
  if (d.ref_start < d.n) {
    k_refactor<<<blocks, 32 * warps, smem, s>>>(d);
    ++*launches;
  }
  return cudaGetLastError();
}

cudaError_t launch_diag_stats(const DevPlan &d, int blocks, cudaStream_t s) {
  if (d.n) k_diag_stats<<<blocks, 256, 0, s>>>(d);
  return cudaGetLastError();
}

}  // namespace kkt
