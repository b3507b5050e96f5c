// Numeric refactorization on the frozen schedule (direct_lu.refactorize, direct_lu.py:297-356).
//
// Persistent warp-per-task kernel, sync-free.  A task is (column, system); tasks are
// dispatched through an atomic ticket in DAG-level order (column-major, system-minor), so
// the chains of all nb systems advance together.  A task's workspace x (the column pattern:
// U rows, diagonal, L rows — sorted positions) lives in shared memory.  The warp replays
// so(j) in the reference's topological order; each update pair carries its precomputed
// workspace slot.
//
// Readiness without flags: every L entry is reset to a sentinel NaN bit pattern before the
// launch, and a consumer re-reads an entry of L(:,k) until it is no longer the sentinel —
// the producer's store of the value is the signal (no fences, one L2 round trip per hop).
// Producers publish L(:,j) before any other bookkeeping.  Update pairs are staged in shared
// memory a chunk at a time with cp.async, two buffers per warp (the next chunk in flight
// while one replays); the sequential replay runs from shared memory.  Products and differences are rounded
// separately (no FMA) and every workspace entry receives its updates in the reference
// order => bitwise equal factors.
#include <cuda_runtime.h>

#include <cstdlib>

#include "device.h"
#include "kernels.cuh"

namespace kkt {

// ----------------------------------------------------------------------------
// Operator values: expand caller layout -> general CSR, inf-norms, max|a| (blockIdx.y =
// system).  One thread per row; sums in entry order (np.bincount order => bitwise).
// ----------------------------------------------------------------------------
constexpr int R_U = 1;  // replay entries per lane in flight

__global__ void __launch_bounds__(256) k_expand_norms(DevPlan d) {
  __shared__ double sh[3][8];
  const int b = blockIdx.y;
  const double *in = d.in_vals + (size_t)b * d.in_cap;
  double *av = d.A_vals + (size_t)b * d.nnz_a;
  double mx = 0.0, sg = 0.0, op = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d.n; i += gridDim.x * blockDim.x) {
    const int rb = d.A_rp[i], s = d.A_split[i], e = d.A_rp[i + 1];
    double g = 0.0, s1 = 0.0, s2 = 0.0;
    for (int p = rb; p < e; ++p) {
      const double v = in[d.sym_lower ? d.gen_src[p] : p];
      av[p] = v;
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
    atomic_max_nonneg(&d.scal[(size_t)b * SCAL_STRIDE + slot], m);
  }
}

__device__ __forceinline__ double patch_floor(const DevPlan &d, int b) {
  // eps_patch = 1e-12 * inf_norm(Ag)                                         (:318)
  return __dmul_rn(PATCH_RELATIVE_FLOOR,
                   __longlong_as_double((long long)d.scal[(size_t)b * SCAL_STRIDE + SC_INFNORM]));
}

// Stage buffers: two per warp, each BUF update-pair values + BUF int slots (template BUF;
// KKT_REF_BUF = 128 | 256 | 512, DevPlan::ref_buf, fixed when the handle is created).

// A chunk of replay steps whose pairs fit a stage buffer (or one step wider than it: big).
struct StChunk {
  int t0, nsteps, npairs, pair0;
  bool big;
  int4 m;     // this lane's step metadata {slot of k, |L(:,k)|, first pair, first L index}
  int incl;   // inclusive prefix of the pair counts
};

template <int BUF>
__device__ __forceinline__ StChunk st_meta(const DevPlan &d, int t0, int t_end, int lane) {
  StChunk c;
  c.t0 = t0;
  const int t = t0 + lane;
  c.m = t < t_end ? d.so_meta[t] : make_int4(0, 0, 0, 0);
  int incl = c.m.y;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  c.incl = incl;
  const unsigned fits = __ballot_sync(0xffffffffu, t < t_end && incl <= BUF);
  c.nsteps = __popc(fits);
  c.big = c.nsteps == 0;  // a single step with more pairs than a stage buffer
  if (c.big) c.nsteps = 1;
  c.pair0 = __shfl_sync(0xffffffffu, c.m.z, 0);
  c.npairs = c.big ? 0 : __shfl_sync(0xffffffffu, incl, c.nsteps - 1);
  return c;
}

// cp.async of a chunk's slots (contiguous int32) and L values (per step a contiguous
// L(:,k)); one commit group per chunk (empty for a big step).
__device__ __forceinline__ void st_issue(const DevPlan &d, const StChunk &c, double *stl, int *sts,
                                         const double *Lx, int lane) {
  if (!c.big) {
    for (int p = lane; p < c.npairs; p += 32) cp_async4(&sts[p], &d.upd_slot32[c.pair0 + p]);
    for (int i = 0; i < c.nsteps; ++i) {
      const int cnt = __shfl_sync(0xffffffffu, c.m.y, i);
      const int off = __shfl_sync(0xffffffffu, c.incl - c.m.y, i);
      const int lbk = __shfl_sync(0xffffffffu, c.m.w, i);
      for (int e = lane; e < cnt; e += 32) cp_async8(&stl[off + e], &Lx[lbk + e]);
    }
  }
  cp_async_commit();
}

template <int BUF>
__global__ void __launch_bounds__(256) k_refactor(DevPlan d) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int wstride = d.maxpat + 3 * BUF;  // doubles per warp: x | 2 x BUF values | 2 x BUF slots
  double *x = smem + (size_t)wib * wstride;
  double *st_l = x + d.maxpat;
  int *st_s = reinterpret_cast<int *>(st_l + 2 * BUF);
  const int ntask = d.ref_n1 * d.nb;  // (single system with wide columns: the light ones only)
  while (true) {
    int task = 0;
    if (lane == 0) task = atomicAdd(d.ticket, 1);
    task = __shfl_sync(0xffffffffu, task, 0);
    if (task >= ntask) break;
    const int sys = task % d.nb;
    const int j = d.col_order[d.ref_start + task / d.nb];
    double *Lx = d.Lx + (size_t)sys * d.nnz_L;
    double *Ux = d.Ux + (size_t)sys * d.nnz_U;
    double *Lv = d.Lv + (size_t)sys * d.nnz_L;
    double *Uv = d.Uv + (size_t)sys * d.nnz_U;
    const double *av = d.A_vals + (size_t)sys * d.nnz_a;
    const bool trace = d.trace_ref && sys == 0;
    if (trace && lane == 0) d.trace_ref[2 * j] = globaltimer();
    const double eps = patch_floor(d, sys);
    const int ub = d.Up[j], nu = d.Up[j + 1] - ub;
    const int lb = d.Lp[j], nl = d.Lp[j + 1] - lb;
    const int np = nu + 1 + nl;
    // for k in so(j) (topological): x[Li(k)] -= Lx(k) * x[k]                  (:324-326)
    // Chunks of steps whose update pairs fit a stage buffer are staged with cp.async, the next
    // chunk's copies in flight while this one replays (two buffers).  L(:,k) is the contiguous
    // Lx[Lp[k], Lp[k+1]) and a chunk's slots are contiguous, so a chunk is one round trip.
    const int t_end = d.so_ptr[j + 1];
    StChunk cur = st_meta<BUF>(d, d.so_ptr[j], t_end, lane);
    st_issue(d, cur, st_l, st_s, Lx, lane);  // in flight during the A scatter
    for (int s = lane; s < np; s += 32) x[s] = 0.0;
    __syncwarp();
    // x[a_tgt] = avals[a_src]                                                 (:323)
    for (int q = d.ap_ptr[j] + lane; q < d.ap_ptr[j + 1]; q += 32) x[d.a_slot[q]] = av[d.a_src[q]];
    __syncwarp();
    int buf = 0;
    while (cur.t0 < t_end) {
      const int tn = cur.t0 + cur.nsteps;
      StChunk nxt;
      nxt.t0 = tn;
      nxt.nsteps = 0;
      if (tn < t_end) {
        nxt = st_meta<BUF>(d, tn, t_end, lane);
        st_issue(d, nxt, st_l + (buf ^ 1) * BUF, st_s + (buf ^ 1) * BUF, Lx, lane);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncwarp();
      double *stl = st_l + buf * BUF;
      const int *sts = st_s + buf * BUF;
      const int nsteps = cur.nsteps, t0 = cur.t0;
      for (int i = 0; i < nsteps; ++i) {
        const int kslot = __shfl_sync(0xffffffffu, cur.m.x, i);
        const int cnt = __shfl_sync(0xffffffffu, cur.m.y, i);
        const int off = __shfl_sync(0xffffffffu, cur.incl - cur.m.y, i);
        const double xk = x[kslot];
        const int lbk = __shfl_sync(0xffffffffu, cur.m.w, i);  // L(:,k) = Lx[lbk, lbk+cnt)
        if (!cur.big) {
          // L(:,k) not yet published when staged?  ref_direct (default): every lane polls its
          // own unpublished entries in the replay below — the values arrive as they are
          // published (10k sequence step 3.75 -> 3.40 ms).  ref_direct 0: one lane waits on the
          // column's last entry, then the whole step is re-staged with one more round trip.
          bool miss = false;
          if (!d.ref_direct)
            for (int e = lane; e < cnt; e += 32) miss |= is_sentinel(stl[off + e]);
          const unsigned mm = __ballot_sync(0xffffffffu, miss);
          if (mm) {
            if (lane == __ffs(mm) - 1) wait_value(&Lx[lbk + cnt - 1], d.poll_ns);
            __syncwarp();
            double lv[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (lane + 32 * q < cnt) lv[q] = ld_relaxed_f64(&Lx[lbk + lane + 32 * q]);
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (lane + 32 * q < cnt) stl[off + lane + 32 * q] = lv[q];
            for (int e = lane + 256; e < cnt; e += 32) stl[off + e] = ld_relaxed_f64(&Lx[lbk + e]);
          }
          // the targets of one step are distinct slots (R_U RMWs per lane in flight;
          // 1 measured fastest: 10k 2.89 ms vs 3.01 with 2, 3.04 with 4)
          for (int e0 = lane; e0 < cnt; e0 += 32 * R_U) {
            double lv[R_U], xv[R_U];
            int sl[R_U];
#pragma unroll
            for (int q = 0; q < R_U; ++q)
              if (e0 + 32 * q < cnt) {
                lv[q] = stl[off + e0 + 32 * q];
                sl[q] = sts[off + e0 + 32 * q];
              }
#pragma unroll
            for (int q = 0; q < R_U; ++q)
              if (e0 + 32 * q < cnt) xv[q] = x[sl[q]];
#pragma unroll
            for (int q = 0; q < R_U; ++q)
              if (e0 + 32 * q < cnt) {
                double l = lv[q];
                if (is_sentinel(l)) l = wait_value(&Lx[lbk + e0 + 32 * q]);  // rare: not yet visible
                x[sl[q]] = __dsub_rn(xv[q], __dmul_rn(l, xk));
              }
          }
          if (d.trace_step && sys == 0 && lane == 0)
            d.trace_step[t0 + i] = globaltimer() | (mm ? 1ull : 0ull);
        } else {  // one step wider than a stage buffer: straight from L2
          const int pair0 = __shfl_sync(0xffffffffu, cur.m.z, i);
          for (int e = lane; e < cnt; e += 32) {
            const double l = wait_value_backoff(&Lx[lbk + e]);
            const int s = d.upd_slot[pair0 + e];
            x[s] = __dsub_rn(x[s], __dmul_rn(l, xk));
          }
        }
        __syncwarp();
      }
      cur = nxt;
      buf ^= 1;
    }
    cp_async_wait<0>();
    __syncwarp();
    // u_jj = x[j]; patch; L(:,j) = x[Li] / u_jj; U(:,j) = x[Ui]                 (:327-344)
    // L(:,j) is what other tasks wait for: publish it first, bookkeeping after.
    double gm = 0.0;
    double ujj = x[nu];
    gm = fmax(gm, fabs(ujj));
    if (fabs(ujj) < eps) {
      ujj = (ujj >= 0.0) ? eps : -eps;
      if (lane == 0) atomicAdd(&d.scal[(size_t)sys * SCAL_STRIDE + SC_PATCHED], 1ull);
    }
    for (int s = lane; s < nl; s += 32) {
      const double v = x[nu + 1 + s];
      gm = fmax(gm, fabs(v));
      const double l = unsentinel(__ddiv_rn(v, ujj));
      st_relaxed_f64(&Lx[lb + s], l);  // value == readiness
      x[nu + 1 + s] = l;               // reused by the CSR copy below (same lane)
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
        if (s < nl) Lv[mp[q]] = x[nu + 1 + s];
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
          Ux[ub + s] = v;
          Uv[mp[q]] = v;
          gm = fmax(gm, fabs(v));
        }
      }
    }
    gm = warp_max(gm);
    if (lane == 0) {
      d.udiag[(size_t)sys * d.n + j] = ujj;
      atomic_max_nonneg(&d.scal[(size_t)sys * SCAL_STRIDE + SC_GMAX], gm);
      if (trace) d.trace_ref[2 * j + 1] = globaltimer();
    }
    __syncwarp();
  }
}

// ----------------------------------------------------------------------------
// Single system, wide columns (j >= JW, the separator tail; second launch): one CTA of
// WIDE_NT threads per column instead of one warp, so a step's |L(:,k)| entries and the
// column's divisions are spread over 256 lanes.  Columns are dispatched by ticket in DAG-level
// order (a column only waits on columns of earlier tickets or of the first launch: deadlock-
// free with any number of resident CTAs).  The column's step metadata is staged in shared
// memory once; each step's L(:,k) values and slots are cp.async'ed WIDE_AHEAD steps ahead into
// a ring of WIDE_AHEAD + 2 slots (the slot written at step t was last read at step t - 2, so
// one barrier per step suffices).  A value staged before it was published is the sentinel and
// is polled in L2 at use.  Steps wider than a ring slot are replayed straight from L2.
// Every workspace entry still receives its updates in so(j) order => bitwise the same factors.
// ----------------------------------------------------------------------------
// CTA width by the tail's mean step size (host: refactor_wide_nt): 10k (36 entries per step)
// 128 threads 1.34 ms vs 256 1.38 vs 512 1.53; imbalance 0.9 (227 per step) 512 10.8 ms vs
// 256 11.9 vs 128 15.5.  Steps staged 3 ahead (2: 1.38, 5: 1.48 ms at 10k).
constexpr int WIDE_AHEAD = 3;
constexpr int WIDE_Q = WIDE_AHEAD + 2;

size_t refactor_wide_smem(int maxpat, int maxsteps, int slot) {
  return ((size_t)maxpat + 1) / 2 * 16 + (size_t)maxsteps * 16 + (size_t)WIDE_Q * slot * 12 + 64;
}

template <int WIDE_NT>
__global__ void __launch_bounds__(WIDE_NT) k_refactor_wide(DevPlan d) {
  extern __shared__ __align__(16) double wsm[];
  __shared__ int s_task;
  __shared__ double s_gm[WIDE_NT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int SL = d.ref_wslot;
  double *x = wsm;                                                              // [maxpat]
  int4 *meta = reinterpret_cast<int4 *>(wsm + ((d.maxpat + 1) & ~1));          // [maxsteps]
  double *rv = reinterpret_cast<double *>(meta + d.ref_wsteps);                 // [Q][SL]
  int *rs = reinterpret_cast<int *>(rv + (size_t)WIDE_Q * SL);                  // [Q][SL]
  const int nw = d.n - d.ref_start - d.ref_n1;
  const double eps = patch_floor(d, 0);
  while (true) {
    if (tid == 0) s_task = atomicAdd(d.ticket2, 1);
    __syncthreads();
    const int task = s_task;
    if (task >= nw) break;
    const int j = d.col_order[d.ref_start + d.ref_n1 + task];
    const int ub = d.Up[j], nu = d.Up[j + 1] - ub;
    const int lb = d.Lp[j], nl = d.Lp[j + 1] - lb;
    const int np = nu + 1 + nl;
    const int t0 = d.so_ptr[j], ns = d.so_ptr[j + 1] - t0;
    for (int t = tid; t < ns; t += WIDE_NT) cp_async16(&meta[t], &d.so_meta[t0 + t]);
    cp_async_commit();
    for (int f = tid; f < np; f += WIDE_NT) x[f] = 0.0;
    __syncthreads();
    // x[a_tgt] = avals[a_src]                                                 (:323)
    for (int q = d.ap_ptr[j] + tid; q < d.ap_ptr[j + 1]; q += WIDE_NT) x[d.a_slot[q]] = d.A_vals[d.a_src[q]];
    cp_async_wait<0>();
    __syncthreads();
    // stage step t into ring slot t % Q (one commit group per step and thread, maybe empty)
    auto issue = [&](int t) {
      if (t < ns) {
        const int4 m = meta[t];  // {slot of k, |L(:,k)|, first pair, first L index}
        if (m.y <= SL) {
          double *v = rv + (size_t)(t % WIDE_Q) * SL;
          int *sl = rs + (size_t)(t % WIDE_Q) * SL;
          for (int e = tid; e < m.y; e += WIDE_NT) {
            cp_async8(&v[e], &d.Lx[m.w + e]);
            cp_async4(&sl[e], &d.upd_slot32[m.z + e]);
          }
        }
      }
      cp_async_commit();
    };
#pragma unroll
    for (int a = 0; a < WIDE_AHEAD; ++a) issue(a);
    // for k in so(j) (topological): x[Li(k)] -= Lx(k) * x[k]                  (:324-326)
    for (int t = 0; t < ns; ++t) {
      issue(t + WIDE_AHEAD);             // into the slot step t - 2 used (finished: barrier)
      cp_async_wait<WIDE_AHEAD>();       // this thread's copies of step t have landed
      __syncthreads();                   // everyone's, and step t - 1's updates of x
      const int4 m = meta[t];
      const double xk = x[m.x];
      if (m.y <= SL) {
        const double *v = rv + (size_t)(t % WIDE_Q) * SL;
        const int *sl = rs + (size_t)(t % WIDE_Q) * SL;
        for (int e = tid; e < m.y; e += WIDE_NT) {
          double l = v[e];
          if (is_sentinel(l)) l = wait_value(&d.Lx[m.w + e], d.poll_ns);  // staged before published
          const int q = sl[e];
          x[q] = __dsub_rn(x[q], __dmul_rn(l, xk));
        }
      } else {  // wider than a ring slot: straight from L2
        for (int e = tid; e < m.y; e += WIDE_NT) {
          const double l = wait_value_backoff(&d.Lx[m.w + e]);
          const int q = d.upd_slot32[m.z + e];
          x[q] = __dsub_rn(x[q], __dmul_rn(l, xk));
        }
      }
    }
    cp_async_wait<0>();
    __syncthreads();
    // u_jj = x[j]; patch; L(:,j) = x[Li] / u_jj (published first); U(:,j) = x[Ui]  (:327-344)
    double ujj = x[nu];
    double gm = fabs(ujj);
    const bool patched = fabs(ujj) < eps;
    if (patched) ujj = (ujj >= 0.0) ? eps : -eps;
    for (int q = tid; q < nl; q += WIDE_NT) {
      const double v = x[nu + 1 + q];
      gm = fmax(gm, fabs(v));
      const double l = unsentinel(__ddiv_rn(v, ujj));
      st_relaxed_f64(&d.Lx[lb + q], l);  // value == readiness
      x[nu + 1 + q] = l;                 // (the same thread rereads it below)
    }
    for (int q = tid; q < nl; q += WIDE_NT) d.Lv[d.Lmap[lb + q]] = x[nu + 1 + q];
    for (int q = tid; q < nu; q += WIDE_NT) {
      const double v = x[q];
      d.Ux[ub + q] = v;
      d.Uv[d.Umap[ub + q]] = v;
      gm = fmax(gm, fabs(v));
    }
    gm = warp_max(gm);
    if (lane == 0) s_gm[warp] = gm;
    __syncthreads();  // also: the workspace is reused by the next task
    if (tid == 0) {
      double g = 0.0;
      for (int w = 0; w < WIDE_NT / 32; ++w) g = fmax(g, s_gm[w]);
      d.udiag[j] = ujj;
      if (patched) atomicAdd(&d.scal[SC_PATCHED], 1ull);
      atomic_max_nonneg(&d.scal[SC_GMAX], g);
    }
  }
}

template <int NT>
static cudaError_t wide_conf(size_t smem, int *blocks_per_sm) {
  cudaError_t e = cudaFuncSetAttribute(k_refactor_wide<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_refactor_wide<NT>, NT, smem);
}
cudaError_t refactor_wide_configure(int nt, size_t smem, int *blocks_per_sm) {
  return nt == 512 ? wide_conf<512>(smem, blocks_per_sm)
         : nt == 128 ? wide_conf<128>(smem, blocks_per_sm) : wide_conf<256>(smem, blocks_per_sm);
}
int refactor_wide_nt(double mean_step) {
  if (const char *e = std::getenv("KKT_REF_WIDE_NT")) {
    const int v = std::atoi(e);
    return v >= 512 ? 512 : v <= 128 ? 128 : 256;
  }
  return mean_step <= 48 ? 128 : mean_step <= 160 ? 256 : 512;  // 70k (54): 256 6.87 vs 128 7.02 ms
}

// ----------------------------------------------------------------------------
// Wide leading levels (level 0: no replay steps; level 1: <= a few) hold most columns but
// almost no work: one thread per (column, system), one launch per level (the kernel
// boundary is the dependency), workspace in local memory.  Same arithmetic as k_refactor.
// ----------------------------------------------------------------------------
constexpr int SMALL_PAT = 64;

constexpr int MAX_BATCH = 64;

__global__ void __launch_bounds__(256) k_refactor_small(DevPlan d, int begin, int end) {
  __shared__ unsigned long long bmax[MAX_BATCH];
  for (int q = threadIdx.x; q < d.nb; q += blockDim.x) bmax[q] = 0ull;
  __syncthreads();
  const int count = end - begin;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int sys = tid / count;  // system-major: a warp mostly serves one system
  const int idx = begin + tid % count;
  double gm = 0.0;
  if (sys < d.nb) {
    const int j = d.col_order[idx];
    double *Lx = d.Lx + (size_t)sys * d.nnz_L;
    const double *av = d.A_vals + (size_t)sys * d.nnz_a;
    const double eps = patch_floor(d, sys);
    const int ub = d.Up[j], nu = d.Up[j + 1] - ub;
    const int lb = d.Lp[j], nl = d.Lp[j + 1] - lb;
    double x[SMALL_PAT];
#pragma unroll 1
    for (int s = 0; s < nu + 1 + nl; ++s) x[s] = 0.0;
    for (int q = d.ap_ptr[j]; q < d.ap_ptr[j + 1]; ++q) x[d.a_slot[q]] = av[d.a_src[q]];
    for (int t = d.so_ptr[j]; t < d.so_ptr[j + 1]; ++t) {
      const int4 m = d.so_meta[t];
      const double xk = x[m.x];
      for (int e = 0; e < m.y; ++e) {
        const int s = d.upd_slot[m.z + e];
        x[s] = __dsub_rn(x[s], __dmul_rn(ldcg(&Lx[m.w + e]), xk));
      }
    }
    double *Ux = d.Ux + (size_t)sys * d.nnz_U;
    double *Uv = d.Uv + (size_t)sys * d.nnz_U;
    double *Lv = d.Lv + (size_t)sys * d.nnz_L;
    for (int s = 0; s < nu; ++s) {
      Ux[ub + s] = x[s];
      Uv[d.Umap[ub + s]] = x[s];
      gm = fmax(gm, fabs(x[s]));
    }
    double ujj = x[nu];
    gm = fmax(gm, fabs(ujj));
    if (fabs(ujj) < eps) {
      ujj = (ujj >= 0.0) ? eps : -eps;
      atomicAdd(&d.scal[(size_t)sys * SCAL_STRIDE + SC_PATCHED], 1ull);
    }
    for (int s = 0; s < nl; ++s) {
      const double v = x[nu + 1 + s];
      gm = fmax(gm, fabs(v));
      const double l = unsentinel(__ddiv_rn(v, ujj));
      Lv[d.Lmap[lb + s]] = l;
      Lx[lb + s] = l;
    }
    d.udiag[(size_t)sys * d.n + j] = ujj;
    if (d.trace_ref && sys == 0) d.trace_ref[2 * j] = d.trace_ref[2 * j + 1] = globaltimer();
    if (gm > 0.0) atomicMax(&bmax[sys], dbits(gm));
  }
  __syncthreads();
  for (int q = threadIdx.x; q < d.nb; q += blockDim.x)
    if (bmax[q]) atomicMax(&d.scal[(size_t)q * SCAL_STRIDE + SC_GMAX], bmax[q]);
}

__global__ void k_diag_stats(DevPlan d) {
  const int b = blockIdx.y;
  const double *ud = d.udiag + (size_t)b * d.n;
  double mx = 0.0, mn = INFINITY;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d.n; i += gridDim.x * blockDim.x) {
    const double a = fabs(ud[i]);
    mx = fmax(mx, a);
    mn = fmin(mn, a);
  }
  mx = warp_max(mx);
  mn = -warp_max(-mn);
  if ((threadIdx.x & 31) == 0) {
    atomic_max_nonneg(&d.scal[(size_t)b * SCAL_STRIDE + SC_MAXPIV], mx);
    if (mn < INFINITY) atomic_min_nonneg(&d.scal[(size_t)b * SCAL_STRIDE + SC_MINPIV], mn);
  }
}

// mode 0: zero the value statistics of every system; mode 1: min |u_jj| := +inf
__global__ void k_reset_scal(unsigned long long *scal, int nb, int mode) {
  for (int q = threadIdx.x; q < nb; q += blockDim.x) {
    unsigned long long *s = scal + (size_t)q * SCAL_STRIDE;
    if (mode == 0) {
      for (int k = 0; k < SC_MINPIV; ++k) s[k] = 0ull;
      s[SC_OPNORM] = 0ull;
    } else {
      s[SC_MINPIV] = 0x7FF0000000000000ull;
    }
  }
}

cudaError_t launch_reset_scal(const DevPlan &d, int mode, cudaStream_t s) {
  k_reset_scal<<<1, 64, 0, s>>>(d.scal, d.nbp, mode);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------
cudaError_t launch_expand_norms(const DevPlan &d, cudaStream_t s) {
  if (d.n) {
    const int bx = min((d.n + 255) / 256, max(1, 2 * 148 / d.nb));
    k_expand_norms<<<dim3(bx, d.nb), 256, 0, s>>>(d);
  }
  return cudaGetLastError();
}

int refactor_buf() {
  const char *e = std::getenv("KKT_REF_BUF");
  const int b = e ? std::atoi(e) : 256;
  return b >= 512 ? 512 : b <= 128 ? 128 : 256;
}

size_t refactor_smem_bytes(int warps, int maxpat, int buf) {
  return (size_t)warps * (maxpat + 3 * buf) * sizeof(double);
}

template <int BUF>
static cudaError_t ref_conf(int warps, size_t smem, int *blocks_per_sm) {
  cudaError_t e = cudaFuncSetAttribute(k_refactor<BUF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(smem > 48 * 1024 ? smem : 48 * 1024));
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, k_refactor<BUF>, 32 * warps, smem);
}

cudaError_t refactor_configure(int warps, size_t smem, int buf, int *blocks_per_sm) {
  return buf == 512 ? ref_conf<512>(warps, smem, blocks_per_sm)
         : buf == 128 ? ref_conf<128>(warps, smem, blocks_per_sm)
                      : ref_conf<256>(warps, smem, blocks_per_sm);
}

cudaError_t launch_refactor(const DevPlan &d, int blocks, int warps, size_t smem, cudaStream_t s,
                            long long *launches) {
  if (!d.n) return cudaSuccess;
  // readiness protocol: L(:,k) entries start as the sentinel
  cudaError_t e = cudaMemsetAsync(d.Lx, 0xFF, 8 * (size_t)d.nnz_L * d.nb, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(d.ticket, 0, 4, s);
  if (e != cudaSuccess) return e;
  // wide leading levels: thread per (column, system), level-synchronous
  for (int l = 0; l < d.n_small_levels; ++l) {
    const int b = d.lev_ptr[l], en = d.lev_ptr[l + 1];
    if (en > b) {
      const long long thr = (long long)(en - b) * d.nb;
      k_refactor_small<<<(unsigned)((thr + 255) / 256), 256, 0, s>>>(d, b, en);
      ++*launches;
    }
  }
  if (d.ref_start < d.n) {
    if (d.ref_buf == 512) k_refactor<512><<<blocks, 32 * warps, smem, s>>>(d);
    else if (d.ref_buf == 128) k_refactor<128><<<blocks, 32 * warps, smem, s>>>(d);
    else k_refactor<256><<<blocks, 32 * warps, smem, s>>>(d);
    ++*launches;
  }
  if (d.ref_start + d.ref_n1 < d.n) {  // single system: the wide columns, CTA per column
    e = cudaMemsetAsync(d.ticket2, 0, 4, s);
    if (e != cudaSuccess) return e;
    if (d.ref_wnt == 512) k_refactor_wide<512><<<d.ref_wblocks, 512, d.ref_wsmem, s>>>(d);
    else if (d.ref_wnt == 128) k_refactor_wide<128><<<d.ref_wblocks, 128, d.ref_wsmem, s>>>(d);
    else k_refactor_wide<256><<<d.ref_wblocks, 256, d.ref_wsmem, s>>>(d);
    ++*launches;
  }
  return cudaGetLastError();
}

cudaError_t launch_diag_stats(const DevPlan &d, int blocks, cudaStream_t s) {
  if (d.n) k_diag_stats<<<dim3(max(1, blocks / d.nb), d.nb), 256, 0, s>>>(d);
  return cudaGetLastError();
}

}  // namespace kkt
