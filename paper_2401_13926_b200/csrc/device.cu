// Host orchestration of the B200 hot path and the C ABI of include/kktb200.h.
//
// Reference behaviour reproduced (pkg/src/kktsolve/...):
//   refactor.cu  k_expand_norms / k_refactor   to_general values + inf_norm, refactorize
//                                              (direct_lu.py:297-356)          bitwise
//   trisolve.cu  k_trsv_grid / k_trsv_cta      lu_solve (direct_lu.py:359-379)  bitwise
//   vector.cu    k_spmv / k_resid_stats        spmv (sparsecore.py:284-305)     bitwise;
//                                              nsr/nrbe/needs_refinement (refine.py:62-92)
//   krylov.cu    k_dots / k_cgs / k_givens ... fgmres + cgs2_step (krylov.py:93-216)
// One handle = one GPU + one stream + one arena allocated at creation (PAPER.md:228:
// "all workspaces preallocated once").
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <new>
#include <queue>
#include <string>
#include <vector>

#include "host_util.h"

namespace kkt {

template <typename S, typename T>
static std::vector<T> narrow(const std::vector<S> &v) {
  std::vector<T> o(v.size());
  for (size_t i = 0; i < v.size(); ++i) o[i] = (T)v[i];
  return o;
}

static std::vector<int> to_i32(const std::vector<int64_t> &v) { return narrow<int64_t, int>(v); }

static int upload(void *dst, const void *src, size_t bytes, cudaStream_t s) {
  if (!bytes) return KKT_OK;
  CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
  return KKT_OK;
}

#define UP(dst, vec) \
  if ((rc = upload(dst, vec.data(), vec.size() * sizeof(vec[0]), dev->stream)) != KKT_OK) return rc

static void destroy(Device *dev) {
  if (!dev) return;
  cudaSetDevice(dev->device);
  if (dev->stream) cudaStreamSynchronize(dev->stream);
  for (Device *hp : dev->helpers) destroy(hp);
  dev->helpers.clear();
  free_krylov(dev);
  if (dev->arena) cudaFree(dev->arena);
  if (dev->trace_mem) cudaFree(dev->trace_mem);
  if (dev->pinned) cudaFreeHost(dev->pinned);
  if (dev->stream) cudaStreamDestroy(dev->stream);
  if (dev->stream2) cudaStreamDestroy(dev->stream2);
  if (dev->ev_a) cudaEventDestroy(dev->ev_a);
  if (dev->ev_b) cudaEventDestroy(dev->ev_b);
  if (dev->ev_h) cudaEventDestroy(dev->ev_h);
  delete dev;
}

// Batched refactor tasks (k_b_refactor): for every column past the thread-per-column levels
// (DAG-level order), chunks of S systems.  S trades coalescing (lanes over systems) against
// the per-column critical path (lanes over entries): the workspace x[np][S] must fit the
// per-warp budget, and heavy columns (many update pairs) get more entry lanes.
// KKT_B_SCHED="lo,mid,hi" overrides the pair thresholds for S <= 8 / 4 / 1.
static int build_batch_tasks(const HostPlan &h, int nbp, int xbudget, int jlo, int jhi,
                             std::vector<int2> &tasks) {
  int lo = 1 << 30, mid = 1 << 30, hi = 1 << 30;  // default: S from the workspace only
  if (const char *e = std::getenv("KKT_B_SCHED")) std::sscanf(e, "%d,%d,%d", &lo, &mid, &hi);
  const int start = h.small_lev_ptr[h.n_small_levels];
  for (int c = start; c < h.n; ++c) {
    const int j = h.col_order[c];
    if (j < jlo || j >= jhi) continue;
    const int64_t np = (h.Up[j + 1] - h.Up[j]) + 1 + (h.Lp[j + 1] - h.Lp[j]);
    if (np > xbudget)
      return set_error(KKT_ERR_BAD_SHAPE, "column pattern too large for the batched workspace");
    int64_t pairs = 0;
    for (int64_t t = h.so_ptr[j]; t < h.so_ptr[j + 1]; ++t) pairs += h.so_meta[4 * t + 1];
    int S = 32;
    while (S > 1 && np * S > xbudget) S >>= 1;
    if (pairs > hi) S = 1;
    else if (pairs > mid) S = std::min(S, 4);
    else if (pairs > lo) S = std::min(S, 8);
    int lg = 0;
    while ((1 << lg) < S) ++lg;
    for (int s0 = 0; s0 < nbp; s0 += S) tasks.push_back(make_int2(j, (s0 << 8) | lg));
  }
  return KKT_OK;
}

// Heavy tail tables (k_b_refactor_heavy): for every column j >= J0 past the thread-per-
// column levels, in DAG-level order: its workspace slots in pull order (U slots in the
// topological so(j) order, the diagonal, the L slots) and, per slot, the updates it
// receives {source slot, L index} in the reference's step order.
struct HeavyPlan {
  std::vector<int> col, optr, pp;
  std::vector<uint16_t> ord;
  std::vector<int2> pairs;
  int xp = 0;
};

static int build_heavy(const HostPlan &h, int J0, HeavyPlan &H) {
  const int start = h.small_lev_ptr[h.n_small_levels];
  H = HeavyPlan();
  H.optr.assign(1, 0);
  H.pp.assign(1, 0);
  std::vector<std::vector<int2>> lists;
  for (int c = start; c < h.n; ++c) {
    const int j = h.col_order[c];
    if (j < J0) continue;
    const int nu = (int)(h.Up[j + 1] - h.Up[j]), nl = (int)(h.Lp[j + 1] - h.Lp[j]);
    const int np = nu + 1 + nl;
    H.col.push_back(j);
    H.xp = std::max(H.xp, np);
    lists.assign(np, {});
    for (int64_t t = h.so_ptr[j]; t < h.so_ptr[j + 1]; ++t) {
      const int k = h.so_data[t], kslot = h.so_slot[t];
      const int64_t p0 = h.upd_ptr[t];
      for (int64_t e = 0; e < h.Lp[k + 1] - h.Lp[k]; ++e)
        lists[h.upd_slot[p0 + e]].push_back(make_int2(kslot, (int)(h.Lp[k] + e)));
    }
    auto emit = [&](int slot) {
      H.ord.push_back((uint16_t)slot);
      H.pairs.insert(H.pairs.end(), lists[slot].begin(), lists[slot].end());
      H.pp.push_back((int)H.pairs.size());
    };
    for (int64_t t = h.so_ptr[j]; t < h.so_ptr[j + 1]; ++t) emit(h.so_slot[t]);
    for (int s = nu; s < np; ++s) emit(s);
    if ((int)H.ord.size() - H.optr.back() != np)
      return set_error(KKT_ERR_BAD_SHAPE, "heavy plan: U pattern and so(j) disagree");
    H.optr.push_back((int)H.ord.size());
  }
  if (H.pairs.size() >= (size_t)INT32_MAX) return set_error(KKT_ERR_BAD_SHAPE, "heavy plan too large");
  return KKT_OK;
}

static int setup(Device *dev, const kkt_device_opts *opts, Device *&out);

static int create(const Symbolic &S, const int64_t *A_rp, const int64_t *A_ci, int64_t in_nnz,
                  const int64_t *gen_src, const kkt_device_opts *opts, Device *&out) {
  out = nullptr;
  Device *dev = new Device();
  int rc = build_plan(S, A_rp, A_ci, in_nnz, gen_src, dev->h);
  if (rc != KKT_OK) {
    delete dev;
    return rc;
  }
  return setup(dev, opts, out);
}

// A handle of another batch width over the same host plan (the straggler helper of a batch).
int create_like(const Device *src, int batch, Device *&out) {
  out = nullptr;
  Device *dev = new Device();
  dev->h = src->h;
  kkt_device_opts o{};
  o.device = src->device;
  o.batch = batch;
  o.restart_m = src->restart_m;
  return setup(dev, &o, out);
}

// Everything after the host plan: device arrays, schedules, launch shapes.
static int setup(Device *dev, const kkt_device_opts *opts, Device *&out) {
  int rc = KKT_OK;
  const HostPlan &h = dev->h;
  dev->device = opts ? opts->device : 0;
  dev->restart_m = (opts && opts->restart_m > 0) ? opts->restart_m : 10;
  const int nb = (opts && opts->batch > 1) ? opts->batch : 1;
  if (nb > 4096) {
    delete dev;
    return set_error(KKT_ERR_BAD_ARG, "batch must be <= 4096");
  }
  const int nbp = nb > 1 ? (nb + 31) / 32 * 32 : 1;  // interleaved width (batch.cu)
  cudaError_t ce = cudaSetDevice(dev->device);
  if (ce == cudaSuccess) ce = cudaStreamCreateWithFlags(&dev->stream, cudaStreamNonBlocking);
  if (ce != cudaSuccess) {
    delete dev;
    return set_error(KKT_ERR_CUDA, std::string("device/stream: ") + cudaGetErrorString(ce));
  }
  cudaDeviceGetAttribute(&dev->sm_count, cudaDevAttrMultiProcessorCount, dev->device);
  DevPlan &d = dev->d;
  d.n = h.n;
  d.nb = nb;
  d.nbp = nbp;
  // reduction blocks per group: the batched vector kernels are HBM-bound, so the grid covers
  // the SMs several times over whatever the number of 32-system groups
  d.rb = nb == 1 ? RED_BLOCKS : std::max(64, 8 * 148 / (nbp / 32));
  std::vector<int2> btask;
  std::vector<int> so_dep;  // wide-column steps: k - J2 for a wide k, else -1 (ct_mode 3)
  HeavyPlan heavy;
  d.b_xbudget = B_XBUDGET;
  d.b_stage = B_STAGE;  // doubles per stage buffer (two buffers per warp)
  d.b_xbudget2 = B_XBUDGET2;
  d.b_stage2 = B_STAGE2;
  if (const char *e = std::getenv("KKT_B_SMEM")) std::sscanf(e, "%d,%d", &d.b_xbudget, &d.b_stage);
  if (const char *e = std::getenv("KKT_B_SMEM2")) std::sscanf(e, "%d,%d", &d.b_xbudget2, &d.b_stage2);
  d.b_static = std::getenv("KKT_B_STATIC") ? std::atoi(std::getenv("KKT_B_STATIC")) : 0;
  d.b_xbudget = (std::max(d.b_xbudget, h.maxpat) + 1) & ~1;  // even: 16-byte pairs (k_b_refactor2)
  d.b_xbudget2 = std::max(d.b_xbudget2, h.maxpat);
  if (nb > 1) {
    // heavy tail: from the first column whose pattern exceeds KKT_B_HEAVY_NP slots
    const int heavy_np = std::getenv("KKT_B_HEAVY_NP") ? std::atoi(std::getenv("KKT_B_HEAVY_NP")) : 0;
    d.J0 = h.n;
    for (int j = 0; j < h.n; ++j)
      if (heavy_np > 0 && (h.Up[j + 1] - h.Up[j]) + 1 + (h.Lp[j + 1] - h.Lp[j]) > heavy_np) {
        d.J0 = j;
        break;
      }
    int rc2 = build_heavy(h, d.J0, heavy);
    if (rc2 == KKT_OK && b_heavy_smem(heavy.xp) > B_HEAVY_SMEM_MAX) {  // too wide for one CTA
      d.J0 = h.n;
      rc2 = build_heavy(h, d.J0, heavy);
    }
    // the replay runs in two launches split at column J2 (first pattern wider than
    // KKT_B_SPLIT_NP slots): warp tasks before it, 4-warp CTA tasks (k_b_refactor_cta) for the
    // wide separator columns after it
    // Default split: 144 slots when the TMA pipeline (ct_mode 3) keeps 3 CTAs per SM for the
    // widest pattern (its replay beats the warp replay from ~144 slots on: 10k 7.28 -> 6.71 ms,
    // 2000 3.13 -> 2.73 ms), else 256 (70k: xp 1351, one CTA per SM, 256 is faster).
    int split_np = 256;
    {
      const int mode = std::getenv("KKT_B_CT_MODE") ? std::atoi(std::getenv("KKT_B_CT_MODE")) : 3;
      const int sc = std::getenv("KKT_B_CT_SC") ? std::atoi(std::getenv("KKT_B_CT_SC")) : 8;
      int maxnp = 1;
      for (int j = 0; j < std::min(d.J0, h.n); ++j)
        maxnp = std::max<int>(maxnp, (int)((h.Up[j + 1] - h.Up[j]) + 1 + (h.Lp[j + 1] - h.Lp[j])));
      int ns = 2, stg = 256;
      b_tma_shape(maxnp, &ns, &stg);
      if (mode == 3 && sc == 8 && b_tma_smem(maxnp, ns, stg) <= 74 * 1024) split_np = 144;
    }
    if (std::getenv("KKT_B_SPLIT_NP")) split_np = std::atoi(std::getenv("KKT_B_SPLIT_NP"));
    int J2 = std::min(d.J0, h.n);
    for (int j = 0; j < J2; ++j)
      if (split_np > 0 && (h.Up[j + 1] - h.Up[j]) + 1 + (h.Lp[j + 1] - h.Lp[j]) > split_np) {
        J2 = j;
        break;
      }
    if (rc2 == KKT_OK) rc2 = build_batch_tasks(h, nbp, d.b_xbudget, 0, J2, btask);
    if (J2 < h.n) {
      d.J2 = J2;
      d.so_dep0 = (int)h.so_ptr[J2];
      so_dep.resize(h.so_data.size() - (size_t)h.so_ptr[J2]);
      for (size_t t = 0; t < so_dep.size(); ++t) {
        const int64_t k = h.so_data[d.so_dep0 + t];
        so_dep[t] = (k >= J2 && k < d.J0) ? (int)(k - J2) : -1;
      }
    }
    d.n_btask1 = (int)btask.size();
    // two systems per lane needs every first-launch task to hold >= 2 systems
    d.b_v2 = std::getenv("KKT_B_V2") ? std::atoi(std::getenv("KKT_B_V2")) : 1;
    if (d.b_stage & 1) d.b_v2 = 0;  // (KKT_B_SMEM override: the stage must hold 16-byte pairs)
    for (int t = 0; d.b_v2 && t < d.n_btask1; ++t)
      if ((btask[t].y & 0xff) == 0) d.b_v2 = 0;
    d.ct_sc = std::getenv("KKT_B_CT_SC") ? std::atoi(std::getenv("KKT_B_CT_SC")) : 8;
    if (d.ct_sc != 2 && d.ct_sc != 8) d.ct_sc = 4;
    d.ct_mode = std::getenv("KKT_B_CT_MODE") ? std::atoi(std::getenv("KKT_B_CT_MODE")) : 3;
    if (d.ct_mode == 3 && (d.ct_sc != 8 || (nbp & 7))) d.ct_mode = 0;  // the TMA pipeline serves 8 systems
    // late steps: 0 staged after the flag; 1 read from L2 after the flag; 2 read from L2 with
    // every value its own readiness flag (no wait on the column flag's release fence)
    d.tma_direct = std::getenv("KKT_B_TMA_DIRECT") ? std::atoi(std::getenv("KKT_B_TMA_DIRECT")) : 2;
    if (rc2 == KKT_OK) {  // k_b_refactor_cta tasks: (column, ct_sc systems)
      // Dispatch order of the wide columns: any topological order is deadlock-free (a task
      // only waits on columns of earlier tickets).  0 (default): level order.
      // KKT_B_TAIL_ORDER=1: critical path first — among the columns whose wide dependencies
      // are all dispatched, the one with the longest remaining chain of update pairs (upward
      // rank) goes next (measured: 10k 6.74 -> 6.99 ms, 2000 2.77 -> 2.73 ms, 70k equal).
      const int lo = std::getenv("KKT_B_TAIL_ORDER") ? std::atoi(std::getenv("KKT_B_TAIL_ORDER")) : 0;
      std::vector<int> order;
      const int J1 = std::min(d.J0, h.n);
      const int start = h.small_lev_ptr[h.n_small_levels];  // columns the small kernel runs
      if (lo == 1 && J2 < J1) {
        const int m = J1 - J2;
        std::vector<char> mine(m, 0);
        for (int c = start; c < h.n; ++c)
          if (h.col_order[c] >= J2 && h.col_order[c] < J1) mine[h.col_order[c] - J2] = 1;
        std::vector<std::vector<int>> succ(m);
        std::vector<int> indeg(m, 0);
        std::vector<int64_t> cost(m, 0), rank(m, 0);
        for (int j = J2; j < J1; ++j) {
          if (!mine[j - J2]) continue;
          for (int64_t t = h.so_ptr[j]; t < h.so_ptr[j + 1]; ++t) {
            const int64_t k = h.so_data[t];
            cost[j - J2] += h.so_meta[4 * t + 1] + 1;
            if (k >= J2 && k < J1 && mine[k - J2]) {
              succ[k - J2].push_back(j - J2);
              ++indeg[j - J2];
            }
          }
        }
        for (int i = m - 1; i >= 0; --i) {  // deps point to smaller columns
          int64_t best = 0;
          for (int q : succ[i]) best = std::max(best, rank[q]);
          rank[i] = cost[i] + best;
        }
        std::priority_queue<std::pair<int64_t, int>> ready;
        for (int i = 0; i < m; ++i)
          if (mine[i] && !indeg[i]) ready.push({rank[i], -i});
        while (!ready.empty()) {
          const int i = -ready.top().second;
          ready.pop();
          order.push_back(J2 + i);
          for (int q : succ[i])
            if (--indeg[q] == 0) ready.push({rank[q], -q});
        }
      } else {
        for (int c = start; c < h.n; ++c)
          if (h.col_order[c] >= J2 && h.col_order[c] < d.J0) order.push_back(h.col_order[c]);
      }
      for (const int j : order) {
        d.h_xp = std::max<int>(d.h_xp, (int)((h.Up[j + 1] - h.Up[j]) + 1 + (h.Lp[j + 1] - h.Lp[j])));
        for (int s0 = 0; s0 < nbp; s0 += d.ct_sc) btask.push_back(make_int2(j, s0 << 8));
      }
    }
    if (rc2 == KKT_OK && btask.size() >= (size_t)INT32_MAX)
      rc2 = set_error(KKT_ERR_BAD_SHAPE, "too many batched tasks");
    if (rc2 != KKT_OK) {
      delete dev;
      return rc2;
    }
  }
  d.n_btask = (int)btask.size();
  d.sym_lower = 0;
  d.has_lower = h.has_lower;
  d.nnz_a = h.nnz_a;
  d.in_nnz = h.in_nnz;
  d.nnz_L = h.nnz_L;
  d.nnz_U = h.nnz_U;
  d.n_so = (int64_t)h.so_data.size();
  d.n_upd = (int64_t)h.upd_slot.size();
  d.n_ap = (int64_t)h.a_src.size();
  d.maxpat = h.maxpat;
  d.n_small_levels = h.n_small_levels;
  for (int l = 0; l <= h.n_small_levels; ++l) d.lev_ptr[l] = h.small_lev_ptr[l];
  d.ref_start = h.small_lev_ptr[h.n_small_levels];
  // Single system: the columns from the first pattern wider than KKT_REF_WIDE_NP slots (the
  // separator tail) go to k_refactor_wide, a CTA per column; col_order past the small levels
  // is uploaded as [warp-kernel columns | wide columns], each part in its level order (a wide
  // column only depends on smaller columns, so the split is a valid kernel boundary).
  d.ref_n1 = h.n - d.ref_start;
  std::vector<int32_t> corder;
  if (nbp == 1) {
    // default split: 128 slots (10k: 64 / 128 / 256 -> 1.32 / 1.33 / 1.42 ms); 256 for the
    // 70k class (6.52 vs 6.87 ms at 128)
    const int wide_np = std::getenv("KKT_REF_WIDE_NP") ? std::atoi(std::getenv("KKT_REF_WIDE_NP"))
                                                       : (h.n > 1000000 ? 256 : 128);
    int JW = h.n;
    for (int j = 0; wide_np > 0 && j < h.n; ++j)
      if ((h.Up[j + 1] - h.Up[j]) + 1 + (h.Lp[j + 1] - h.Lp[j]) > wide_np) {
        JW = j;
        break;
      }
    if (JW < h.n) {
      std::vector<int32_t> light, wide;
      int maxsteps = 0, maxcnt = 0;
      int64_t wsteps = 0, wpairs = 0;
      for (int c = d.ref_start; c < h.n; ++c) {
        const int j = h.col_order[c];
        if (j < JW) {
          light.push_back(j);
          continue;
        }
        wide.push_back(j);
        maxsteps = std::max<int>(maxsteps, (int)(h.so_ptr[j + 1] - h.so_ptr[j]));
        for (int64_t t = h.so_ptr[j]; t < h.so_ptr[j + 1]; ++t) {
          maxcnt = std::max<int>(maxcnt, h.so_meta[4 * t + 1]);
          wpairs += h.so_meta[4 * t + 1];
          ++wsteps;
        }
      }
      const int slot = std::max(1, std::min(maxcnt, 1024));  // wider steps: straight from L2
      const size_t smem = refactor_wide_smem(h.maxpat, maxsteps, slot);
      if (!wide.empty() && smem <= 200 * 1024) {
        corder.assign(h.col_order.begin(), h.col_order.begin() + d.ref_start);
        corder.insert(corder.end(), light.begin(), light.end());
        corder.insert(corder.end(), wide.begin(), wide.end());
        d.ref_n1 = (int)light.size();
        d.ref_wslot = slot;
        d.ref_wsteps = maxsteps;
        d.ref_wsmem = smem;
        d.ref_wnt = refactor_wide_nt(wsteps ? (double)wpairs / (double)wsteps : 0.0);
      }
    }
  }
  d.poll_ns = std::getenv("KKT_POLL_NS") ? std::atoi(std::getenv("KKT_POLL_NS")) : (nbp > 1 ? 64 : 0);
  // single system: one lane waits on the critical dependency before the row (without it the
  // lanes poll their unpublished columns at once: 1.27 -> 3.16 ms at 10k); batch: no up-front
  // wait (the lanes are systems, one 256-byte line per poll: 3.62 -> 1.84 ms at 10k x 64)
  d.grid_wait = std::getenv("KKT_GRID_WAIT") ? std::atoi(std::getenv("KKT_GRID_WAIT")) : (nbp > 1 ? 0 : 1);
  d.pL = h.pL;
  d.pU = h.pU;
  d.nLg = (int)h.L_grid_order.size();
  d.L_nsync = (int)h.L_sync_ptr.size() - 1;
  for (int l = 0; l <= d.L_nsync; ++l) d.L_sync_ptr[l] = h.L_sync_ptr[l];
  d.nUg = (int)h.U_grid_order.size();
  d.sweep_maxL = h.sweep_maxL;
  d.sweep_maxU = h.sweep_maxU;
  const size_t n = (size_t)h.n, B = (size_t)nbp;
  {
    const size_t biggest = std::max<size_t>({(size_t)h.nnz_a, (size_t)h.nnz_L, (size_t)h.nnz_U, n + 1});
    if (biggest * B >= ((size_t)1 << 32)) {
      destroy(dev);
      return set_error(KKT_ERR_BAD_SHAPE, "batch too large: interleaved arrays exceed 2^32 elements");
    }
  }
  const size_t in_cap = (size_t)std::max(d.in_nnz, d.nnz_a);
  d.in_cap = (int64_t)in_cap;
  size_t bytes = 0;
  auto acc = [&](size_t b) { bytes += align_up(b + 1); };
  acc(4 * (n + 1)); acc(4 * d.nnz_a); acc(4 * n); acc(4 * d.nnz_a);  // A_rp ci split gen_src
  acc(8 * in_cap * nb); acc(8 * d.nnz_a * B);                        // in_vals A_vals
  if (nbp > 1) acc(8 * in_cap * B);                                    // in_il
  acc(4 * (n + 1)); acc(4 * (n + 1)); acc(4 * d.n_ap); acc(4 * n);   // so_ptr ap_ptr a_src order
  acc(4 * (n + 1)); acc(4 * (n + 1)); acc(4 * d.nnz_L); acc(4 * d.nnz_U);  // Lp Up Lmap Umap
  acc(4 * d.n_upd); acc(16 * d.n_so); acc(2 * d.n_upd); acc(2 * d.n_ap);   // lidx meta slots
  acc(8 * d.nnz_L * B); acc(8 * d.nnz_U * B); acc(8 * n * B);              // Lx Ux udiag
  acc(4 * (n + 1)); acc(4 * d.nnz_L); acc(4 * (n + 1)); acc(4 * d.nnz_U);  // Lrp Lci Urp Uci
  acc(4 * n); acc(4 * n);                                                  // perms
  acc(4 * h.L_grid_order.size()); acc(4 * h.L_tail_order.size());
  acc(4 * h.U_head_order.size()); acc(4 * h.U_grid_order.size());
  acc(4 * h.L_crit.size()); acc(4 * h.U_crit.size()); acc(4 * h.Uhead_off.size());
  acc(4 * d.nnz_L); acc(4 * d.nnz_U);                                      // Li Ui (CSC)
  acc(4 * h.Ltail_split.size()); acc(8 * h.Ltail_split.size() * B);        // split, tacc
  acc(4 * h.Ugrid_split.size()); acc(4 * h.U_part_rows.size());            // U head prefix
  acc(4 * h.Lc_task.size()); acc(4 * h.Lc_aux.size()); acc(4 * h.Lc_split.size());  // chains
  acc(4 * h.Uc_task.size()); acc(4 * h.Uc_aux.size()); acc(4 * h.Uc_split.size());
  if (nbp == 1) acc(8 * n);                                                // cpart
  acc(8 * d.nnz_L * B); acc(8 * d.nnz_U * B); acc(8 * n * B); acc(8 * n * B);  // Lv Uv yL yU
  acc(8 * SCAL_STRIDE * B); acc(64); acc(8 * 8 * (size_t)d.rb * B);        // scal ticket partials
  acc(8 * btask.size());                                                   // batched tasks
  acc(4 * h.L_glev_ptr.size()); acc(4 * h.U_glev_ptr.size()); acc(64);     // levels, barrier
  acc(4 * heavy.col.size()); acc(4 * heavy.optr.size()); acc(4 * heavy.pp.size());
  acc(2 * heavy.ord.size()); acc(8 * heavy.pairs.size()); acc(64);          // heavy tail
  const size_t ncflag = d.J2 < n ? (size_t)(n - d.J2) * (size_t)(nbp / 8 + 1) : 0;
  acc(4 * so_dep.size()); acc(4 * ncflag);                                 // wide-column flags
  for (const HostSweep *hs : {&h.swL, &h.swU}) {
    acc(4 * hs->dptr.size()); acc(4 * hs->dsrc.size()); acc(2 * hs->ddst.size());
    acc(4 * hs->dmask.size()); acc(4 * hs->bptr.size()); acc(4 * hs->brow.size());
    acc(4 * hs->bbeg.size()); acc(4 * hs->bcnt.size()); acc(4 * hs->bofs.size());
  }
  ce = cudaMalloc(&dev->arena, bytes);
  if (ce != cudaSuccess) {
    destroy(dev);
    return set_error(KKT_ERR_OOM, "cudaMalloc of the device plan failed");
  }
  dev->arena_bytes = bytes;
  char *cur = (char *)dev->arena;
  d.A_rp = carve<int>(cur, n + 1);
  d.A_ci = carve<int>(cur, d.nnz_a);
  d.A_split = carve<int>(cur, n);
  d.gen_src = carve<int>(cur, d.nnz_a);
  d.in_vals = carve<double>(cur, in_cap * nb);
  if (nbp > 1) d.in_il = carve<double>(cur, in_cap * B);
  d.A_vals = carve<double>(cur, d.nnz_a * B);
  d.so_ptr = carve<int>(cur, n + 1);
  d.ap_ptr = carve<int>(cur, n + 1);
  d.a_src = carve<int>(cur, d.n_ap);
  d.col_order = carve<int>(cur, n);
  d.Lp = carve<int>(cur, n + 1);
  d.Up = carve<int>(cur, n + 1);
  d.Lmap = carve<int>(cur, d.nnz_L);
  d.Umap = carve<int>(cur, d.nnz_U);
  d.upd_lidx = carve<int>(cur, d.n_upd);
  d.so_meta = carve<int4>(cur, d.n_so);
  d.upd_slot = carve<uint16_t>(cur, d.n_upd);
  d.a_slot = carve<uint16_t>(cur, d.n_ap);
  d.Lx = carve<double>(cur, d.nnz_L * B);
  d.Ux = carve<double>(cur, d.nnz_U * B);
  d.udiag = carve<double>(cur, n * B);
  d.Lrp = carve<int>(cur, n + 1);
  d.Lci = carve<int>(cur, d.nnz_L);
  d.Urp = carve<int>(cur, n + 1);
  d.Uci = carve<int>(cur, d.nnz_U);
  d.row_perm = carve<int>(cur, n);
  d.col_perm = carve<int>(cur, n);
  d.L_grid_order = carve<int>(cur, h.L_grid_order.size());
  d.L_tail_order = carve<int>(cur, h.L_tail_order.size());
  d.U_head_order = carve<int>(cur, h.U_head_order.size());
  d.U_grid_order = carve<int>(cur, h.U_grid_order.size());
  d.L_crit = carve<int>(cur, h.L_crit.size());
  d.U_crit = carve<int>(cur, h.U_crit.size());
  d.Uhead_off = carve<int>(cur, h.Uhead_off.size());
  d.Li = carve<int>(cur, d.nnz_L);
  d.Ui = carve<int>(cur, d.nnz_U);
  d.Ltail_split = carve<int>(cur, h.Ltail_split.size());
  d.tacc = carve<double>(cur, h.Ltail_split.size() * B);
  d.Ugrid_split = carve<int>(cur, h.Ugrid_split.size());
  d.U_part_rows = carve<int>(cur, h.U_part_rows.size());
  d.n_upart = (int)h.U_part_rows.size();
  d.u_partial = std::getenv("KKT_U_PARTIAL") ? std::atoi(std::getenv("KKT_U_PARTIAL")) : 1;
  d.Lc_task = carve<int>(cur, h.Lc_task.size());
  d.Lc_aux = carve<int>(cur, h.Lc_aux.size());
  d.Lc_split = carve<int>(cur, h.Lc_split.size());
  d.Uc_task = carve<int>(cur, h.Uc_task.size());
  d.Uc_aux = carve<int>(cur, h.Uc_aux.size());
  d.Uc_split = carve<int>(cur, h.Uc_split.size());
  d.nLc = (int)h.Lc_task.size();
  d.nUc = (int)h.Uc_task.size();
  if (nbp == 1) d.cpart = carve<double>(cur, n);
  // chain tasks: single system, U grid rows starting at their head split (the plan's model)
  d.chains = (nbp == 1 && d.u_partial && (d.nLc > 0 || d.nUc > 0)) ? 1 : 0;
  if (std::getenv("KKT_CHAINS")) d.chains = d.chains && std::atoi(std::getenv("KKT_CHAINS")) != 0;
  d.Lv = carve<double>(cur, d.nnz_L * B);
  d.Uv = carve<double>(cur, d.nnz_U * B);
  d.yL = carve<double>(cur, n * B);
  d.yU = carve<double>(cur, n * B);
  d.scal = carve<unsigned long long>(cur, SCAL_STRIDE * B);
  d.ticket = carve<int>(cur, 16);
  d.partials = carve<double>(cur, 8 * (size_t)d.rb * B);
  d.btask = carve<int2>(cur, btask.size());
  d.L_glev = carve<int>(cur, h.L_glev_ptr.size());
  d.U_glev = carve<int>(cur, h.U_glev_ptr.size());
  d.gbar = carve<unsigned>(cur, 16);
  d.L_nglev = (int)h.L_glev_ptr.size() - 1;
  d.U_nglev = (int)h.U_glev_ptr.size() - 1;
  d.b_levelsync = std::getenv("KKT_B_LEVELSYNC") ? std::atoi(std::getenv("KKT_B_LEVELSYNC")) : 0;
  d.nhc = (int)heavy.col.size();
  d.h_xp = std::max(d.h_xp, heavy.xp);
  d.hc_col = carve<int>(cur, heavy.col.size());
  d.hc_optr = carve<int>(cur, heavy.optr.size());
  d.h_pp = carve<int>(cur, heavy.pp.size());
  d.h_ord = carve<uint16_t>(cur, heavy.ord.size());
  d.h_pairs = carve<int2>(cur, heavy.pairs.size());
  d.ticket2 = carve<int>(cur, 16);
  d.so_dep = carve<int>(cur, so_dep.size());
  d.cflag = carve<int>(cur, ncflag);
  {
    const HostSweep *hs[2] = {&h.swL, &h.swU};
    SweepDev *sd[2] = {&d.swL, &d.swU};
    for (int k = 0; k < 2; ++k) {
      sd[k]->nblk = hs[k]->nblk;
      sd[k]->dptr = carve<int>(cur, hs[k]->dptr.size());
      sd[k]->dsrc = carve<int>(cur, hs[k]->dsrc.size());
      sd[k]->ddst = carve<uint16_t>(cur, hs[k]->ddst.size());
      sd[k]->dmask = carve<unsigned>(cur, hs[k]->dmask.size());
      sd[k]->bptr = carve<int>(cur, hs[k]->bptr.size());
      sd[k]->brow = carve<int>(cur, hs[k]->brow.size());
      sd[k]->bbeg = carve<int>(cur, hs[k]->bbeg.size());
      sd[k]->bcnt = carve<int>(cur, hs[k]->bcnt.size());
      sd[k]->bofs = carve<int>(cur, hs[k]->bofs.size());
      sd[k]->max_stage = hs[k]->max_stage;
    }
  }
  d.trace_ref = d.trace_trsv = d.trace_step = nullptr;
  if (std::getenv("KKT_TRACE") && std::atoi(std::getenv("KKT_TRACE")) > 0) {
    const size_t tb = 4 * 8 * n + 8 * std::max<size_t>((size_t)d.n_so, 4 * n);
    ce = cudaMalloc(&dev->trace_mem, tb + 64);
    if (ce == cudaSuccess) {
      d.trace_ref = (unsigned long long *)dev->trace_mem;
      d.trace_trsv = d.trace_ref + 2 * n;
      d.trace_step = d.trace_trsv + 2 * n;
      if (std::atoi(std::getenv("KKT_TRACE")) == 2) d.trace_trsv = nullptr;  // chain loop cycles only
      cudaMemsetAsync(dev->trace_mem, 0, tb, dev->stream);
    }
  }
  UP(d.A_rp, to_i32(h.A_rp));
  UP(d.A_ci, to_i32(h.A_ci));
  UP(d.A_split, to_i32(h.A_split));
  UP(d.gen_src, to_i32(h.gen_src));
  UP(d.so_ptr, to_i32(h.so_ptr));
  UP(d.ap_ptr, to_i32(h.ap_ptr));
  UP(d.a_src, h.a_src);
  if (corder.empty()) {
    UP(d.col_order, h.col_order);
  } else {
    UP(d.col_order, corder);
  }
  UP(d.Lp, to_i32(h.Lp));
  UP(d.Up, to_i32(h.Up));
  UP(d.Lmap, h.Lmap);
  UP(d.Umap, h.Umap);
  {  // the replays derive L indices from the step metadata (L(:,k) is contiguous in Lx); the
     // buffer holds int32 slots for their cp.async staging
    d.upd_slot32 = d.upd_lidx;
    d.upd_lidx = nullptr;
    const std::vector<int> slot32 = narrow<uint16_t, int>(h.upd_slot);
    UP(d.upd_slot32, slot32);
  }
  UP(d.so_meta, h.so_meta);
  UP(d.upd_slot, h.upd_slot);
  UP(d.a_slot, h.a_slot);
  UP(d.Lrp, h.Lrp);
  UP(d.Lci, h.Lci);
  UP(d.Urp, h.Urp);
  UP(d.Uci, h.Uci);
  UP(d.row_perm, to_i32(h.row_perm));
  UP(d.col_perm, to_i32(h.col_perm));
  UP(d.L_grid_order, h.L_grid_order);
  UP(d.L_tail_order, h.L_tail_order);
  UP(d.U_head_order, h.U_head_order);
  UP(d.U_grid_order, h.U_grid_order);
  UP(d.L_crit, h.L_crit);
  UP(d.U_crit, h.U_crit);
  UP(d.Uhead_off, h.Uhead_off);
  UP(d.Li, h.Li32);
  UP(d.Ui, h.Ui32);
  UP(d.Ltail_split, h.Ltail_split);
  UP(d.Ugrid_split, h.Ugrid_split);
  UP(d.U_part_rows, h.U_part_rows);
  UP(d.Lc_task, h.Lc_task);
  UP(d.Lc_aux, h.Lc_aux);
  UP(d.Lc_split, h.Lc_split);
  UP(d.Uc_task, h.Uc_task);
  UP(d.Uc_aux, h.Uc_aux);
  UP(d.Uc_split, h.Uc_split);
  UP(d.btask, btask);
  UP(d.so_dep, so_dep);
  UP(d.hc_col, heavy.col);
  UP(d.hc_optr, heavy.optr);
  UP(d.h_pp, heavy.pp);
  UP(d.h_ord, heavy.ord);
  UP(d.h_pairs, heavy.pairs);
  UP(d.L_glev, h.L_glev_ptr);
  UP(d.U_glev, h.U_glev_ptr);
  CUDA_TRY(cudaMemsetAsync(d.gbar, 0, 64, dev->stream));
  UP(d.swL.dptr, h.swL.dptr); UP(d.swL.dsrc, h.swL.dsrc); UP(d.swL.ddst, h.swL.ddst);
  UP(d.swL.dmask, h.swL.dmask); UP(d.swL.bptr, h.swL.bptr); UP(d.swL.brow, h.swL.brow);
  UP(d.swL.bbeg, h.swL.bbeg); UP(d.swL.bcnt, h.swL.bcnt); UP(d.swL.bofs, h.swL.bofs);
  UP(d.swU.dptr, h.swU.dptr); UP(d.swU.dsrc, h.swU.dsrc); UP(d.swU.ddst, h.swU.ddst);
  UP(d.swU.dmask, h.swU.dmask); UP(d.swU.bptr, h.swU.bptr); UP(d.swU.brow, h.swU.brow);
  UP(d.swU.bbeg, h.swU.bbeg); UP(d.swU.bcnt, h.swU.bcnt); UP(d.swU.bofs, h.swU.bofs);
  // the first factorization's values, so solve() works before any refactor (LuFactors);
  // a batch starts every system from them (broadcast into the interleaved layout)
  {
    std::vector<double> lv(h.nnz_L), uv(h.nnz_U);
    for (int64_t p = 0; p < h.nnz_L; ++p) lv[h.Lmap[p]] = h.Lx0[p];
    for (int64_t p = 0; p < h.nnz_U; ++p) uv[h.Umap[p]] = h.Ux0[p];
    if (nbp == 1) {
      UP(d.Lx, h.Lx0);
      UP(d.Ux, h.Ux0);
      UP(d.udiag, h.Udiag0);
      UP(d.Lv, lv);
      UP(d.Uv, uv);
      CUDA_TRY(cudaStreamSynchronize(dev->stream));
    } else {
      const size_t mx = std::max<size_t>({(size_t)h.nnz_L, (size_t)h.nnz_U, n, 1});
      double *tmp = nullptr;
      ce = cudaMalloc(&tmp, 8 * mx);
      if (ce != cudaSuccess) {
        destroy(dev);
        return set_error(KKT_ERR_OOM, "cudaMalloc of the upload buffer failed");
      }
      struct Arr { const std::vector<double> *v; double *dst; } arrs[5] = {
          {&h.Lx0, d.Lx}, {&h.Ux0, d.Ux}, {&h.Udiag0, d.udiag}, {&lv, d.Lv}, {&uv, d.Uv}};
      for (auto &a : arrs) {
        if (a.v->empty()) continue;
        ce = cudaMemcpyAsync(tmp, a.v->data(), 8 * a.v->size(), cudaMemcpyHostToDevice, dev->stream);
        if (ce == cudaSuccess) ce = b_launch_broadcast(tmp, (int64_t)a.v->size(), nbp, a.dst, dev->stream);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(dev->stream);
        if (ce != cudaSuccess) break;
      }
      cudaFree(tmp);
      if (ce != cudaSuccess) {
        destroy(dev);
        return set_error(KKT_ERR_CUDA, std::string("initial factors: ") + cudaGetErrorString(ce));
      }
    }
  }
  CUDA_TRY(launch_fill_sentinel(d.yL, (int64_t)(n * B), dev->stream));
  CUDA_TRY(launch_fill_sentinel(d.yU, (int64_t)(n * B), dev->stream));
  if (d.cpart) CUDA_TRY(launch_fill_sentinel(d.cpart, (int64_t)n, dev->stream));
  CUDA_TRY(cudaMemsetAsync(d.scal, 0, 8 * SCAL_STRIDE * B, dev->stream));
  CUDA_TRY(cudaMemsetAsync(d.ticket, 0, 64, dev->stream));
  // launch shapes
  CUDA_TRY(sweep_configure());
  if (nbp > 1) {
    int rbps = 0, tbps = 0;
    dev->refactor_smem = b_refactor_smem(d.b_xbudget, d.b_stage);
    if (d.ct_mode == 3) {
      b_tma_shape(std::max(d.h_xp, 1), &d.tma_ns, &d.tma_stg);
      // KKT_B_TMA_E=64: 16 consumer warps per CTA (measured at 70k, one CTA per SM: 96.6 ->
      // 98.0 ms, so 32 entry lanes stay the default everywhere)
      d.tma_e = std::getenv("KKT_B_TMA_E") ? std::atoi(std::getenv("KKT_B_TMA_E")) : 32;
      if (d.tma_e == 64) {
        d.tma_ns = 2;
        d.tma_stg = 256;
      } else {
        d.tma_e = 32;
      }
      // flag-free producer where the stage ring was cut to 128 rows (wide patterns, one or
      // two CTAs per SM: batch.cu k_b_refactor_tma FLAGS)
      if (!std::getenv("KKT_B_TMA_DIRECT")) d.tma_direct = (d.tma_e == 32 && d.tma_stg == 128) ? 3 : 2;
    }
    const size_t smem2 = d.ct_mode == 3 ? b_tma_smem(std::max(d.h_xp, 1), d.tma_ns, d.tma_stg)
                                        : b_cta_smem(std::max(d.h_xp, 1), d.ct_sc);
    int rbps2 = 0;
    d.b_gridv = b_grid_variant();
    CUDA_TRY(b_configure(nbp, dev->refactor_smem, d.b_gridv, &rbps, &tbps));
    if (d.ct_mode == 3) {
      CUDA_TRY(b_tma_configure(d.tma_ns, d.tma_stg, d.tma_e, d.tma_direct != 3, smem2, &rbps2));
      CUDA_TRY(b_tma_maps(d));
    } else {
      CUDA_TRY(b_cta_configure(d.ct_sc, smem2, &rbps2, d.ct_mode == 2));
    }
    dev->refactor_blocks2 = std::max(1, rbps2) * dev->sm_count;
    dev->refactor_smem2 = smem2;
    // overlapped launches (KKT_B_OVERLAP=1; measured slower): one wide-column CTA per SM next to
    // as many warp-replay CTAs as still fit
    const int ov = std::getenv("KKT_B_OVERLAP") ? std::atoi(std::getenv("KKT_B_OVERLAP")) : 0;
    if (ov && rbps2 >= 1 && d.ct_mode != 3) {  // (the TMA pipeline needs phase 1 complete)
      cudaDeviceProp prop;
      CUDA_TRY(cudaGetDeviceProperties(&prop, dev->device));
      const size_t sm_left = prop.sharedMemPerMultiprocessor - smem2 - prop.reservedSharedMemPerBlock;
      const int fit = (int)(sm_left / (dev->refactor_smem + prop.reservedSharedMemPerBlock));
      const int b1 = std::min(std::max(rbps, 1), fit);
      if (b1 >= 1) {
        dev->refactor_blocks_ov = b1 * dev->sm_count;
        dev->refactor_blocks2 = dev->sm_count;  // one wide-column CTA per SM
        CUDA_TRY(cudaStreamCreateWithFlags(&dev->stream2, cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&dev->ev_a, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&dev->ev_b, cudaEventDisableTiming));
      }
    }
    dev->refactor_warps = B_WARPS;
    if (d.trace_step) d.prof = d.trace_step;  // per-warp cycle counters
    dev->refactor_blocks = std::max(1, rbps) * dev->sm_count;
    dev->trsv_blocks = std::max(1, tbps) * dev->sm_count;
    // residual statistics + scalar blocks of every system (dev_residual_norms, refactor diag)
    dev->pinned_bytes = std::max<size_t>(64 * 1024, 8 * (5 + SCAL_STRIDE) * (size_t)nbp + 4096);
    CUDA_TRY(cudaMallocHost(&dev->pinned, dev->pinned_bytes));
    rc = alloc_krylov(dev, dev->restart_m);
    if (rc != KKT_OK) return rc;
    CUDA_TRY(cudaStreamSynchronize(dev->stream));
    out = dev;
    return KKT_OK;
  }
  dev->refactor_warps = 8;
  d.ref_buf = refactor_buf();
  d.ref_direct = std::getenv("KKT_REF_DIRECT") ? std::atoi(std::getenv("KKT_REF_DIRECT")) : 1;
  dev->refactor_smem = refactor_smem_bytes(dev->refactor_warps, d.maxpat, d.ref_buf);
  while (dev->refactor_smem > 200 * 1024 && dev->refactor_warps > 1) {
    dev->refactor_warps /= 2;
    dev->refactor_smem = refactor_smem_bytes(dev->refactor_warps, d.maxpat, d.ref_buf);
  }
  if (dev->refactor_smem > 220 * 1024) {
    destroy(dev);
    return set_error(KKT_ERR_BAD_SHAPE, "column pattern too large for the shared-memory workspace");
  }
  int bps = 0;
  CUDA_TRY(refactor_configure(dev->refactor_warps, dev->refactor_smem, d.ref_buf, &bps));
  dev->refactor_blocks = std::max(1, bps) * dev->sm_count;
  if (d.ref_start + d.ref_n1 < n) {
    int wb = 0;
    CUDA_TRY(refactor_wide_configure(d.ref_wnt, d.ref_wsmem, &wb));
    d.ref_wblocks = std::max(1, wb) * dev->sm_count;
  }
  int tb = 0;
  CUDA_TRY(trsv_configure(&tb));
  dev->trsv_blocks = std::max(1, tb) * dev->sm_count;
  if (const char *e = std::getenv("KKT_TRSV_BLOCKS")) dev->trsv_blocks = std::max(1, std::atoi(e));
  dev->trsv_blocks_full = dev->trsv_blocks;
  dev->pinned_bytes = 64 * 1024;
  CUDA_TRY(cudaMallocHost(&dev->pinned, dev->pinned_bytes));
  rc = alloc_krylov(dev, dev->restart_m);
  if (rc != KKT_OK) return rc;
  CUDA_TRY(cudaStreamSynchronize(dev->stream));
  out = dev;
  return KKT_OK;
}

static int set_values(Device *dev, const double *vals, int layout, int on_device) {
  DevPlan &d = dev->d;
  if (layout == KKT_LAYOUT_SYMMETRIC_LOWER && !d.has_lower)
    return set_error(KKT_ERR_BAD_ARG, "handle was created without the symmetric-lower map");
  if (layout != KKT_LAYOUT_GENERAL && layout != KKT_LAYOUT_SYMMETRIC_LOWER)
    return set_error(KKT_ERR_BAD_ARG, "unknown value layout");
  d.sym_lower = layout == KKT_LAYOUT_SYMMETRIC_LOWER ? 1 : 0;
  const int64_t cnt = d.sym_lower ? d.in_nnz : d.nnz_a;
  // values_in is [nb][cnt]; the device copy has a per-system pitch of in_cap
  if (d.nbp > 1) {  // batched: transpose straight from the caller's device values
    const double *src = vals;
    if (!on_device) {
      CUDA_TRY(cudaMemcpyAsync(d.in_vals, vals, 8 * (size_t)cnt * d.nb, cudaMemcpyHostToDevice, dev->stream));
      src = d.in_vals;
    }
    LAUNCH(b_launch_transpose(d, src, cnt, d.in_il, dev->stream));
  } else {
    CUDA_TRY(cudaMemcpy2DAsync(d.in_vals, 8 * (size_t)d.in_cap, vals, 8 * (size_t)cnt, 8 * (size_t)cnt,
                               (size_t)d.nb, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                               dev->stream));
  }
  LAUNCH(launch_reset_scal(d, 0, dev->stream));
  LAUNCH(d.nbp > 1 ? b_launch_expand_norms(d, dev->stream) : launch_expand_norms(d, dev->stream));
  return KKT_OK;
}

static int refactor(Device *dev, const double *vals, int layout, int on_device, double *diag_out) {
  DevPlan &d = dev->d;
  int rc = set_values(dev, vals, layout, on_device);
  if (rc != KKT_OK) return rc;
  LAUNCH(launch_reset_scal(d, 1, dev->stream));  // min |u_jj| starts at +inf
  {
    cudaError_t e = d.nbp > 1
                        ? b_launch_refactor(d, dev->refactor_blocks, dev->refactor_smem,
                                            dev->refactor_blocks2, dev->refactor_smem2, dev->stream,
                                            &dev->launches, dev->stream2, dev->ev_a, dev->ev_b,
                                            dev->refactor_blocks_ov)
                        : launch_refactor(d, dev->refactor_blocks, dev->refactor_warps,
                                          dev->refactor_smem, dev->stream, &dev->launches);
    if (e != cudaSuccess) return set_error(KKT_ERR_CUDA, std::string("refactor: ") + cudaGetErrorString(e));
  }
  LAUNCH(d.nbp > 1 ? b_launch_diag_stats(d, dev->stream) : launch_diag_stats(d, dev->sm_count, dev->stream));
  if (diag_out) {  // [nb][4] = {max|u|, min|u|, patched, growth}
    CUDA_TRY(cudaMemcpyAsync(dev->pinned, d.scal, 8 * SCAL_STRIDE * (size_t)d.nb, cudaMemcpyDeviceToHost,
                             dev->stream));
    CUDA_TRY(cudaStreamSynchronize(dev->stream));
    for (int q = 0; q < d.nb; ++q) {
      unsigned long long s[SC_COUNT];
      std::memcpy(s, dev->pinned + (size_t)q * SCAL_STRIDE, sizeof s);
      double v[SC_COUNT];
      std::memcpy(v, s, sizeof v);
      double *o = diag_out + 4 * q;
      o[0] = v[SC_MAXPIV];
      o[1] = d.n ? v[SC_MINPIV] : 0.0;
      o[2] = (double)s[SC_PATCHED];
      o[3] = v[SC_MAXABS_A] > 0 ? v[SC_GMAX] / v[SC_MAXABS_A] : 0.0;
    }
  }
  return KKT_OK;
}

int dev_solve(Device *dev, const double *b, double *x) {
  cudaError_t e = dev->d.nbp > 1 ? b_launch_trsv(dev->d, b, x, dev->trsv_blocks, dev->stream, &dev->launches)
                                 : launch_trsv(dev->d, b, x, dev->trsv_blocks, dev->stream, &dev->launches);
  if (e != cudaSuccess) return set_error(KKT_ERR_CUDA, std::string("trisolve: ") + cudaGetErrorString(e));
  return KKT_OK;
}

int dev_spmv(Device *dev, const double *x, double *y, const double *bsub, double *nrm_partials) {
  LAUNCH(dev->d.nbp > 1 ? b_launch_spmv(dev->d, x, y, bsub, nrm_partials, dev->stream)
                        : launch_spmv(dev->d, x, y, bsub, nrm_partials, dev->stream));
  return KKT_OK;
}

// out6 [nb][6] = {||r-Kx||_2, ||r-Kx||_inf, ||x||_2, ||x||_inf, ||r||_2, ||K||_inf}
int dev_residual_norms(Device *dev, const double *r, const double *x, double *out6) {
  DevPlan &d = dev->d;
  const size_t nb = (size_t)d.nb;
  if (8 * (5 + SCAL_STRIDE) * nb > dev->pinned_bytes)
    return set_error(KKT_ERR_BAD_ARG, "residual statistics exceed the pinned staging buffer");
  double *out5 = d.partials + 5 * (size_t)d.rb * d.nbp;  // after the [nbp][5][rb] partials
  LAUNCH(d.nbp > 1 ? b_launch_resid_stats(d, r, x, d.partials, out5, dev->stream)
                   : launch_resid_stats(d, r, x, d.partials, out5, dev->stream));
  dev->launches++;
  CUDA_TRY(cudaMemcpyAsync(dev->pinned, out5, 8 * 5 * nb, cudaMemcpyDeviceToHost, dev->stream));
  CUDA_TRY(cudaMemcpyAsync(dev->pinned + 5 * nb, d.scal, 8 * SCAL_STRIDE * nb, cudaMemcpyDeviceToHost,
                           dev->stream));
  CUDA_TRY(cudaStreamSynchronize(dev->stream));
  for (size_t q = 0; q < nb; ++q) {
    std::memcpy(out6 + 6 * q, dev->pinned + 5 * q, 5 * 8);
    std::memcpy(out6 + 6 * q + 5, dev->pinned + 5 * nb + q * SCAL_STRIDE + SC_OPNORM, 8);
  }
  return KKT_OK;
}

// ---------------------------------------------------------------------------
// Standalone operator handle (struct Operator, host_util.h)
// ---------------------------------------------------------------------------
static int op_create(int64_t n, const int64_t *rp, const int64_t *ci, int sym, int device,
                     Operator *&out) {
  out = nullptr;
  if (n < 0 || n >= INT32_MAX / 2) return set_error(KKT_ERR_BAD_SHAPE, "bad operator dimension");
  const int64_t nnz = rp[n];
  // general pattern + source map (the value-moving half of to_general, sparsecore.py:263)
  std::vector<int64_t> grp(n + 1, 0), gci, src;
  if (sym) {
    for (int64_t i = 0; i < n; ++i)
      for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
        if (ci[p] > i) return set_error(KKT_ERR_BAD_SHAPE, "entry above diagonal in symmetric-lower storage");
        grp[i + 1]++;
        if (ci[p] != i) grp[ci[p] + 1]++;
      }
    for (int64_t i = 0; i < n; ++i) grp[i + 1] += grp[i];
    gci.resize(grp[n]);
    src.resize(grp[n]);
    std::vector<int64_t> fill(grp.begin(), grp.end() - 1);
    // row-major sweep: row i gets its lower entries (cols ascending <= i) ...
    // ... and mirrored entries (i, k) for k > i arrive in ascending k => sorted rows.
    for (int64_t i = 0; i < n; ++i)
      for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
        int64_t q = fill[i]++;
        gci[q] = ci[p];
        src[q] = p;
      }
    for (int64_t i = 0; i < n; ++i)
      for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
        if (ci[p] != i) {
          int64_t q = fill[ci[p]]++;
          gci[q] = i;
          src[q] = p;
        }
    // rows now hold [lower part ascending][mirrored part ascending] = ascending overall
  } else {
    grp.assign(rp, rp + n + 1);
    gci.assign(ci, ci + nnz);
    src.resize(nnz);
    for (int64_t e = 0; e < nnz; ++e) src[e] = e;
  }
  const int64_t ng = grp[n];
  if (ng >= INT32_MAX) return set_error(KKT_ERR_BAD_SHAPE, "operator too large");
  std::vector<int> split(n);
  for (int64_t i = 0; i < n; ++i) {
    int64_t p = grp[i];
    while (p < grp[i + 1] && gci[p] <= i) ++p;
    split[i] = (int)p;
  }
  Operator *op = new Operator();
  op->device = device;
  cudaError_t ce = cudaSetDevice(device);
  if (ce == cudaSuccess) ce = cudaStreamCreateWithFlags(&op->stream, cudaStreamNonBlocking);
  if (ce != cudaSuccess) {
    delete op;
    return set_error(KKT_ERR_CUDA, std::string("operator stream: ") + cudaGetErrorString(ce));
  }
  DevPlan &d = op->d;
  d.n = (int)n;
  d.nnz_a = ng;
  d.in_nnz = nnz;
  d.in_cap = std::max(nnz, ng);
  d.sym_lower = sym ? 1 : 0;
  d.has_lower = sym ? 1 : 0;
  size_t bytes = 0;
  auto acc = [&](size_t b) { bytes += align_up(b + 1); };
  acc(4 * (n + 1)); acc(4 * ng); acc(4 * n); acc(4 * ng); acc(8 * std::max(nnz, ng)); acc(8 * ng);
  acc(8 * 32); acc(8 * 8 * RED_BLOCKS);
  ce = cudaMalloc(&op->arena, bytes);
  if (ce != cudaSuccess) {
    cudaStreamDestroy(op->stream);
    delete op;
    return set_error(KKT_ERR_OOM, "cudaMalloc of the operator failed");
  }
  char *cur = (char *)op->arena;
  d.A_rp = carve<int>(cur, n + 1);
  d.A_ci = carve<int>(cur, ng);
  d.A_split = carve<int>(cur, n);
  d.gen_src = carve<int>(cur, ng);
  d.in_vals = carve<double>(cur, std::max(nnz, ng));
  d.A_vals = carve<double>(cur, ng);
  d.scal = carve<unsigned long long>(cur, 32);
  d.partials = carve<double>(cur, 8 * RED_BLOCKS);
  std::vector<int> a = narrow<int64_t, int>(grp), b = narrow<int64_t, int>(gci), c = narrow<int64_t, int>(src);
  cudaMemcpyAsync(d.A_rp, a.data(), 4 * a.size(), cudaMemcpyHostToDevice, op->stream);
  cudaMemcpyAsync(d.A_ci, b.data(), 4 * b.size(), cudaMemcpyHostToDevice, op->stream);
  cudaMemcpyAsync(d.A_split, split.data(), 4 * split.size(), cudaMemcpyHostToDevice, op->stream);
  cudaMemcpyAsync(d.gen_src, c.data(), 4 * c.size(), cudaMemcpyHostToDevice, op->stream);
  cudaMemsetAsync(d.scal, 0, 8 * 32, op->stream);
  ce = cudaMallocHost(&op->pinned, 4096);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(op->stream);
  if (ce != cudaSuccess) {
    cudaFree(op->arena);
    cudaStreamDestroy(op->stream);
    delete op;
    return set_error(KKT_ERR_CUDA, std::string("operator upload: ") + cudaGetErrorString(ce));
  }
  out = op;
  return KKT_OK;
}

}  // namespace kkt

// ============================================================================
// C ABI
// ============================================================================
using kkt::Device;

extern "C" {

int kkt_dev_create(const kkt_symbolic *s, const int64_t *A_row_ptr, const int64_t *A_col_idx,
                   int64_t in_nnz, const int64_t *gen_src, const kkt_device_opts *opts,
                   kkt_device **out) {
  if (!s || !out || !A_row_ptr || !A_col_idx) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  *out = nullptr;
  try {
    Device *dev = nullptr;
    int rc = kkt::create(*reinterpret_cast<const kkt::Symbolic *>(s), A_row_ptr, A_col_idx, in_nnz,
                         gen_src, opts, dev);
    if (rc != KKT_OK) return rc;
    if ((rc = kkt::prepare_helpers(dev)) != KKT_OK) {
      kkt::destroy(dev);
      return rc;
    }
    *out = reinterpret_cast<kkt_device *>(dev);
    return KKT_OK;
  } catch (std::bad_alloc &) {
    return kkt::set_error(KKT_ERR_OOM, "host allocation failed in kkt_dev_create");
  }
}

int kkt_plan_check(const kkt_symbolic *s, const int64_t *A_row_ptr, const int64_t *A_col_idx,
                   int64_t in_nnz, const int64_t *gen_src, int64_t out[8]) {
  if (!s || !out || !A_row_ptr || !A_col_idx) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  try {
    kkt::HostPlan P;
    const int rc = kkt::build_plan(*reinterpret_cast<const kkt::Symbolic *>(s), A_row_ptr, A_col_idx, in_nnz,
                                   gen_src, P);
    if (rc != KKT_OK) return rc;
    kkt::check_chains(P, out);
    return KKT_OK;
  } catch (std::bad_alloc &) {
    return kkt::set_error(KKT_ERR_OOM, "host allocation failed in kkt_plan_check");
  }
}

void kkt_dev_destroy(kkt_device *d) { kkt::destroy(reinterpret_cast<Device *>(d)); }

void *kkt_dev_stream(kkt_device *d) { return d ? (void *)reinterpret_cast<Device *>(d)->stream : nullptr; }

int kkt_dev_refactor(kkt_device *d, const double *values_in, int layout, int values_on_device,
                     double *diag_out) {
  Device *dev = reinterpret_cast<Device *>(d);
  if (!dev || !values_in) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(dev->device);
  return kkt::refactor(dev, values_in, layout, values_on_device, diag_out);
}

int kkt_dev_set_operator_values(kkt_device *d, const double *values_in, int layout,
                                int values_on_device) {
  Device *dev = reinterpret_cast<Device *>(d);
  if (!dev || !values_in) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(dev->device);
  return kkt::set_values(dev, values_in, layout, values_on_device);
}

int kkt_dev_download_factors(kkt_device *d, double *Lx, double *Ux, double *Udiag) {
  Device *dev = reinterpret_cast<Device *>(d);
  if (!dev) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(dev->device);
  const kkt::DevPlan &p = dev->d;
  const size_t nb = (size_t)p.nb;
  cudaStream_t s = dev->stream;
  cudaError_t e = cudaSuccess;
  if (p.nbp > 1) {  // interleaved [entry][nbp] -> caller [nb][entry]
    const size_t nbp = (size_t)p.nbp;
    struct Arr { const double *src; double *dst; size_t cnt; } arrs[3] = {
        {p.Lx, Lx, (size_t)p.nnz_L}, {p.Ux, Ux, (size_t)p.nnz_U}, {p.udiag, Udiag, (size_t)p.n}};
    for (auto &a : arrs) {
      if (!a.dst || !a.cnt) continue;
      std::vector<double> tmp(a.cnt * nbp);
      e = cudaMemcpyAsync(tmp.data(), a.src, 8 * tmp.size(), cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) return kkt::set_error(KKT_ERR_CUDA, cudaGetErrorString(e));
      for (size_t q = 0; q < nb; ++q)
        for (size_t i = 0; i < a.cnt; ++i) a.dst[q * a.cnt + i] = tmp[i * nbp + q];
    }
    return KKT_OK;
  }
  if (Lx && p.nnz_L) e = cudaMemcpyAsync(Lx, p.Lx, 8 * (size_t)p.nnz_L * nb, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && Ux && p.nnz_U)
    e = cudaMemcpyAsync(Ux, p.Ux, 8 * (size_t)p.nnz_U * nb, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && Udiag && p.n)
    e = cudaMemcpyAsync(Udiag, p.udiag, 8 * (size_t)p.n * nb, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return kkt::set_error(KKT_ERR_CUDA, cudaGetErrorString(e));
  return KKT_OK;
}

int kkt_dev_upload_factors(kkt_device *d, const double *Lx, const double *Ux, const double *Udiag) {
  Device *dev = reinterpret_cast<Device *>(d);
  if (!dev || !Lx || !Ux || !Udiag) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  if (dev->d.nbp != 1) return kkt::set_error(KKT_ERR_BAD_ARG, "kkt_dev_upload_factors needs batch == 1");
  cudaSetDevice(dev->device);
  const kkt::HostPlan &h = dev->h;
  const kkt::DevPlan &p = dev->d;
  // both layouts: CSC (the refactor's) and CSR (the solves'), through the CSC->CSR maps
  std::vector<double> lv(h.nnz_L), uv(h.nnz_U);
  for (int64_t q = 0; q < h.nnz_L; ++q) lv[h.Lmap[q]] = Lx[q];
  for (int64_t q = 0; q < h.nnz_U; ++q) uv[h.Umap[q]] = Ux[q];
  cudaStream_t s = dev->stream;
  cudaError_t e = cudaSuccess;
  if (h.nnz_L) e = cudaMemcpyAsync(p.Lx, Lx, 8 * (size_t)h.nnz_L, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && h.nnz_L) e = cudaMemcpyAsync(p.Lv, lv.data(), 8 * lv.size(), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && h.nnz_U) e = cudaMemcpyAsync(p.Ux, Ux, 8 * (size_t)h.nnz_U, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && h.nnz_U) e = cudaMemcpyAsync(p.Uv, uv.data(), 8 * uv.size(), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && p.n) e = cudaMemcpyAsync(p.udiag, Udiag, 8 * (size_t)p.n, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return kkt::set_error(KKT_ERR_CUDA, cudaGetErrorString(e));
  return KKT_OK;
}

// Batched handles keep vectors interleaved internally; the ABI takes [nb][n] and converts
// through the handle's staging vectors.
#define IL_IN(src, dst)                                                                   \
  do {                                                                                    \
    cudaError_t _e = kkt::b_launch_to_il(dev->d, src, dst, dev->stream);                  \
    dev->launches++;                                                                      \
    if (_e != cudaSuccess) return kkt::set_error(KKT_ERR_CUDA, cudaGetErrorString(_e));   \
  } while (0)
#define IL_OUT(src, dst)                                                                  \
  do {                                                                                    \
    cudaError_t _e = kkt::b_launch_from_il(dev->d, src, dst, dev->stream);                \
    dev->launches++;                                                                      \
    if (_e != cudaSuccess) return kkt::set_error(KKT_ERR_CUDA, cudaGetErrorString(_e));   \
  } while (0)

int kkt_dev_solve(kkt_device *d, const double *b_dev, double *x_dev) {
  Device *dev = reinterpret_cast<Device *>(d);
  if (!dev || !b_dev || !x_dev) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(dev->device);
  if (dev->d.nbp > 1) {
    IL_IN(b_dev, dev->kry->w);
    int rc = kkt::dev_solve(dev, dev->kry->w, dev->kry->w1);
    if (rc) return rc;
    IL_OUT(dev->kry->w1, x_dev);
    return KKT_OK;
  }
  return kkt::dev_solve(dev, b_dev, x_dev);
}

// The kernels alone, on vectors in the handle's internal layout ([n][nbp] interleaved for a
// batch): what bench.py times for the per-kernel roofline (no boundary transposes).
int kkt_dev_solve_native(kkt_device *d, const double *b_dev, double *x_dev) {
  Device *dev = reinterpret_cast<Device *>(d);
  if (!dev || !b_dev || !x_dev) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(dev->device);
  return kkt::dev_solve(dev, b_dev, x_dev);
}

int kkt_dev_spmv_native(kkt_device *d, const double *x_dev, double *y_dev) {
  Device *dev = reinterpret_cast<Device *>(d);
  if (!dev || !x_dev || !y_dev) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(dev->device);
  return kkt::dev_spmv(dev, x_dev, y_dev, nullptr, nullptr);
}

int kkt_dev_spmv(kkt_device *d, const double *x_dev, double *y_dev) {
  Device *dev = reinterpret_cast<Device *>(d);
  if (!dev || !x_dev || !y_dev) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(dev->device);
  if (dev->d.nbp > 1) {
    IL_IN(x_dev, dev->kry->w);
    int rc = kkt::dev_spmv(dev, dev->kry->w, dev->kry->w1, nullptr, nullptr);
    if (rc) return rc;
    IL_OUT(dev->kry->w1, y_dev);
    return KKT_OK;
  }
  return kkt::dev_spmv(dev, x_dev, y_dev, nullptr, nullptr);
}

int kkt_dev_residual(kkt_device *d, const double *r_dev, const double *x_dev, double *rho_dev,
                     double *norms_host) {
  Device *dev = reinterpret_cast<Device *>(d);
  if (!dev || !r_dev || !x_dev || !rho_dev || !norms_host)
    return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(dev->device);
  kkt::DevPlan &p = dev->d;
  const double *r = r_dev, *x = x_dev;
  double *rho = rho_dev;
  if (p.nbp > 1) {  // interleave through the staging vectors
    IL_IN(r_dev, dev->kry->sr);
    IL_IN(x_dev, dev->kry->sx0);
    r = dev->kry->sr;
    x = dev->kry->sx0;
    rho = dev->kry->sx;
  }
  int rc = kkt::dev_spmv(dev, x, rho, r, p.partials);  // rho = r - K x, ||rho||^2 partials
  if (rc) return rc;
  {
    cudaError_t e = kkt::launch_reduce_partials(p, p.partials, 1, dev->kry->nrm, 1, 1, dev->stream);
    dev->launches++;
    if (e != cudaSuccess) return kkt::set_error(KKT_ERR_CUDA, cudaGetErrorString(e));
  }
  if (p.nbp > 1) IL_OUT(rho, rho_dev);
  cudaError_t e = cudaMemcpyAsync(norms_host, dev->kry->nrm, 8 * (size_t)p.nb, cudaMemcpyDeviceToHost,
                                  dev->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(dev->stream);
  if (e != cudaSuccess) return kkt::set_error(KKT_ERR_CUDA, cudaGetErrorString(e));
  return KKT_OK;
}

int kkt_dev_axpy(kkt_device *d, double *x_dev, const double *y_dev) {
  Device *dev = reinterpret_cast<Device *>(d);
  if (!dev || !x_dev || !y_dev) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(dev->device);
  cudaError_t e = kkt::launch_add_inplace(x_dev, y_dev, (int64_t)dev->d.n * dev->d.nb, dev->stream);
  dev->launches++;
  if (e != cudaSuccess) return kkt::set_error(KKT_ERR_CUDA, cudaGetErrorString(e));
  return KKT_OK;
}

int kkt_dev_residual_norms(kkt_device *d, const double *r_dev, const double *x_dev, double *out_host) {
  Device *dev = reinterpret_cast<Device *>(d);
  if (!dev || !r_dev || !x_dev || !out_host) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(dev->device);
  if (dev->d.nbp > 1) {
    IL_IN(r_dev, dev->kry->w);
    IL_IN(x_dev, dev->kry->w1);
    return kkt::dev_residual_norms(dev, dev->kry->w, dev->kry->w1, out_host);
  }
  return kkt::dev_residual_norms(dev, r_dev, x_dev, out_host);
}

int kkt_dev_fgmres(kkt_device *d, const double *b_dev, const double *x0_dev, double *x_dev,
                   const kkt_krylov_cfg *cfg, kkt_krylov_report *rep, double *history_host, int hist_cap) {
  return kkt_dev_fgmres_ops(d, nullptr, nullptr, b_dev, x0_dev, x_dev, cfg, rep, history_host, hist_cap,
                            nullptr, 0);
}

int kkt_dev_fgmres_ops(kkt_device *d, const kkt_linop *K, const kkt_linop *M, const double *b_dev,
                       const double *x0_dev, double *x_dev, const kkt_krylov_cfg *cfg,
                       kkt_krylov_report *rep, double *history_host, int hist_cap,
                       double *restart_pairs_host, int pairs_cap) {
  Device *dev = reinterpret_cast<Device *>(d);
  if (!dev || !b_dev || !x0_dev || !x_dev || !cfg || !rep)
    return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  for (const kkt_linop *op : {K, M}) {
    if (!op) continue;
    if (op->kind < KKT_OP_HANDLE || op->kind > KKT_OP_CALLBACK)
      return kkt::set_error(KKT_ERR_BAD_ARG, "unknown operator kind");
    if (op->kind == KKT_OP_MATRIX &&
        (!op->matrix || reinterpret_cast<kkt::Operator *>(op->matrix)->d.n != dev->d.n))
      return kkt::set_error(KKT_ERR_BAD_ARG, "matrix operator missing or of the wrong dimension");
    if (op->kind == KKT_OP_CALLBACK && !op->apply) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL callback");
  }
  cudaSetDevice(dev->device);
  int rc = kkt::ensure_krylov(dev, cfg->m);  // before staging into the workspace
  if (rc) return rc;
  if (dev->d.nbp > 1) {
    kkt::Krylov &Kr = *dev->kry;
    IL_IN(b_dev, Kr.sr);
    IL_IN(x0_dev, Kr.sx0);
    rc = kkt::dev_fgmres(dev, Kr.sr, Kr.sx0, Kr.sx, cfg, 0, nullptr, K, M, rep, history_host, hist_cap,
                         restart_pairs_host, pairs_cap);
    if (rc && rc != KKT_ERR_NONFINITE) return rc;
    IL_OUT(Kr.sx, x_dev);
    return rc;
  }
  return kkt::dev_fgmres(dev, b_dev, x0_dev, x_dev, cfg, 0, nullptr, K, M, rep, history_host, hist_cap,
                         restart_pairs_host, pairs_cap);
}

// refine_fgmres for every system of the handle (refine.py:103-132): the per-system trigger
// ||r - K x0||_2 > delta ||r||_2, FGMRES(tol = delta) on the triggered systems and x0 for the
// others, all decided on the device (one graph, one host sync).  Vectors in the handle's
// native layout.
static int refine_native(Device *dev, const double *r_dev, const double *x0_dev, double *x_dev,
                         const kkt_krylov_cfg *cfg, kkt_krylov_report *rep,
                         const std::function<int()> *post = nullptr) {
  if (!(cfg->delta_tol > 0) && !cfg->delta_sys) return kkt::set_error(KKT_ERR_BAD_ARG, "delta_tol must be positive");
  return kkt::dev_fgmres(dev, r_dev, x0_dev, x_dev, cfg, 1, nullptr, nullptr, nullptr, rep, nullptr, 0,
                         nullptr, 0, post);
}

int kkt_dev_refine_fgmres(kkt_device *d, const double *r_dev, const double *x0_dev, double *x_dev,
                          const kkt_krylov_cfg *cfg, kkt_krylov_report *rep) {
  Device *dev = reinterpret_cast<Device *>(d);
  if (!dev || !r_dev || !x0_dev || !x_dev || !cfg || !rep)
    return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(dev->device);
  int rc = kkt::ensure_krylov(dev, cfg->m);
  if (rc) return rc;
  if (dev->d.nbp > 1) {
    kkt::Krylov &K = *dev->kry;
    IL_IN(r_dev, K.sr);
    IL_IN(x0_dev, K.sx0);
    rc = refine_native(dev, K.sr, K.sx0, K.sx, cfg, rep);
    if (rc && rc != KKT_ERR_NONFINITE) return rc;
    IL_OUT(K.sx, x_dev);
    return rc;
  }
  return refine_native(dev, r_dev, x0_dev, x_dev, cfg, rep);
}

int kkt_dev_step(kkt_device *d, const double *values_in, int layout, const double *r_in,
                 double *x_out, int io_on_device, const kkt_krylov_cfg *cfg, kkt_krylov_report *rep,
                 double *diag_out) {
  Device *dev = reinterpret_cast<Device *>(d);
  if (!dev || !values_in || !r_in || !x_out || !cfg || !rep)
    return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(dev->device);
  int rc = kkt::refactor(dev, values_in, layout, io_on_device, diag_out);
  if (rc) return rc;
  return kkt_dev_step_solve(d, r_in, x_out, io_on_device, cfg, rep);
}

int kkt_dev_step_solve(kkt_device *d, const double *r_in, double *x_out, int io_on_device,
                       const kkt_krylov_cfg *cfg, kkt_krylov_report *rep) {
  Device *dev = reinterpret_cast<Device *>(d);
  if (!dev || !r_in || !x_out || !cfg || !rep) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(dev->device);
  int rc = kkt::ensure_krylov(dev, cfg->m);  // before staging into the workspace
  if (rc) return rc;
  kkt::Krylov &K = *dev->kry;
  const bool il = dev->d.nbp > 1;
  const size_t bytes = 8 * (size_t)dev->d.n * dev->d.nb;  // caller layout [nb][n]
  const double *r_dev = r_in;
  cudaError_t e = cudaSuccess;
  if (!io_on_device) {  // H2D into the (system-major) staging vector
    double *dst = il ? K.w : K.sr;
    e = cudaMemcpyAsync(dst, r_in, bytes, cudaMemcpyHostToDevice, dev->stream);
    if (e != cudaSuccess) return kkt::set_error(KKT_ERR_CUDA, cudaGetErrorString(e));
    r_dev = dst;
  }
  if (il) {
    IL_IN(r_dev, K.sr);
    r_dev = K.sr;
  }
  rc = kkt::dev_solve(dev, r_dev, K.sx0);  // x0 = lu_solve(r)      (harness.py:234)
  if (rc) return rc;
  // x out of the workspace (caller layout, host or device), enqueued behind the FGMRES graph
  // so the whole step synchronises once (again after a straggler hand-off)
  const std::function<int()> post = [&]() -> int {
    const double *xs = K.sx;
    if (il) {  // (staging in w1: a straggler hand-off after this reads the batch's w)
      double *dst = io_on_device ? x_out : K.w1;
      IL_OUT(K.sx, dst);
      xs = dst;
    }
    if (xs != x_out) {
      cudaError_t ce = cudaMemcpyAsync(x_out, xs, bytes,
                                       io_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                       dev->stream);
      if (ce != cudaSuccess) return kkt::set_error(KKT_ERR_CUDA, cudaGetErrorString(ce));
    }
    return KKT_OK;
  };
  rc = refine_native(dev, r_dev, K.sx0, K.sx, cfg, rep, &post);  // (harness.py:240)
  if (rc && rc != KKT_ERR_NONFINITE) return rc;
  return rc;  // per-system failures (NONFINITE) still return every x
}

int kkt_op_create(int64_t n, const int64_t *row_ptr, const int64_t *col_idx, int symmetric_lower,
                  int device, kkt_operator **out) {
  if (!row_ptr || !out || (n > 0 && !col_idx)) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  *out = nullptr;
  try {
    kkt::Operator *op = nullptr;
    int rc = kkt::op_create(n, row_ptr, col_idx, symmetric_lower, device, op);
    if (rc) return rc;
    *out = reinterpret_cast<kkt_operator *>(op);
    return KKT_OK;
  } catch (std::bad_alloc &) {
    return kkt::set_error(KKT_ERR_OOM, "host allocation failed in kkt_op_create");
  }
}

void kkt_op_destroy(kkt_operator *o) {
  kkt::Operator *op = reinterpret_cast<kkt::Operator *>(o);
  if (!op) return;
  cudaSetDevice(op->device);
  cudaStreamSynchronize(op->stream);
  cudaFree(op->arena);
  cudaFreeHost(op->pinned);
  cudaStreamDestroy(op->stream);
  delete op;
}

void *kkt_op_stream(kkt_operator *o) {
  return o ? (void *)reinterpret_cast<kkt::Operator *>(o)->stream : nullptr;
}

// The operator shares the kernels of the device handle through a lightweight Device view.
static kkt::Device op_view(kkt::Operator *op) {
  kkt::Device v;
  v.device = op->device;
  v.stream = op->stream;
  v.d = op->d;
  v.pinned = op->pinned;
  v.pinned_bytes = 4096;
  return v;
}

int kkt_op_set_values(kkt_operator *o, const double *values, int on_device) {
  kkt::Operator *op = reinterpret_cast<kkt::Operator *>(o);
  if (!op || !values) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(op->device);
  kkt::Device v = op_view(op);
  int rc = kkt::set_values(&v, values, op->d.has_lower ? KKT_LAYOUT_SYMMETRIC_LOWER : KKT_LAYOUT_GENERAL,
                           on_device);
  op->launches += v.launches;
  v.stream = nullptr;
  v.pinned = nullptr;
  return rc;
}

int kkt_op_spmv(kkt_operator *o, const double *x_dev, double *y_dev) {
  kkt::Operator *op = reinterpret_cast<kkt::Operator *>(o);
  if (!op || !x_dev || !y_dev) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(op->device);
  kkt::Device v = op_view(op);
  int rc = kkt::dev_spmv(&v, x_dev, y_dev, nullptr, nullptr);
  op->launches += v.launches;
  v.stream = nullptr;
  v.pinned = nullptr;
  return rc;
}

int kkt_op_residual_norms(kkt_operator *o, const double *r_dev, const double *x_dev, double *out_host) {
  kkt::Operator *op = reinterpret_cast<kkt::Operator *>(o);
  if (!op || !r_dev || !x_dev || !out_host) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  cudaSetDevice(op->device);
  kkt::Device v = op_view(op);
  int rc = kkt::dev_residual_norms(&v, r_dev, x_dev, out_host);
  op->launches += v.launches;
  v.stream = nullptr;
  v.pinned = nullptr;
  return rc;
}

int kkt_dev_info(kkt_device *dd, int64_t info[16]) {
  Device *dev = reinterpret_cast<Device *>(dd);
  if (!dev || !info) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  const kkt::HostPlan &h = dev->h;
  const int64_t v[16] = {h.n, h.pL, h.pU, h.L_grid_levels, h.U_grid_levels, h.n - h.pL, h.n - h.pU,
                         dev->refactor_blocks, dev->refactor_warps, (int64_t)dev->refactor_smem,
                         dev->trsv_blocks, h.refactor_levels, (int64_t)dev->arena_bytes,
                         (int64_t)h.upd_slot.size(), 0, 0};
  for (int i = 0; i < 16; ++i) info[i] = v[i];
  return KKT_OK;
}

int kkt_dev_trace_steps(kkt_device *dd, uint64_t *steps_out) {
  Device *dev = reinterpret_cast<Device *>(dd);
  if (!dev || !dev->d.trace_step) return kkt::set_error(KKT_ERR_BAD_ARG, "tracing disabled");
  cudaSetDevice(dev->device);
  cudaError_t e = cudaStreamSynchronize(dev->stream);
  if (e == cudaSuccess)
    e = cudaMemcpy(steps_out, dev->d.trace_step,
                   8 * std::max<size_t>((size_t)dev->d.n_so, 4 * (size_t)dev->d.n), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return kkt::set_error(KKT_ERR_CUDA, cudaGetErrorString(e));
  return KKT_OK;
}

int kkt_dev_trace(kkt_device *dd, uint64_t *refactor_out, uint64_t *trisolve_out) {
  Device *dev = reinterpret_cast<Device *>(dd);
  if (!dev) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL argument");
  if (!dev->d.trace_ref) return kkt::set_error(KKT_ERR_BAD_ARG, "tracing disabled (set KKT_TRACE=1)");
  cudaSetDevice(dev->device);
  const size_t n = (size_t)dev->d.n;
  cudaError_t e = cudaStreamSynchronize(dev->stream);
  if (e == cudaSuccess && refactor_out)
    e = cudaMemcpy(refactor_out, dev->d.trace_ref, 16 * n, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && trisolve_out)
    e = cudaMemcpy(trisolve_out, dev->d.trace_trsv, 16 * n, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return kkt::set_error(KKT_ERR_CUDA, cudaGetErrorString(e));
  return KKT_OK;
}

int64_t kkt_dev_launch_count(kkt_device *d) {
  return d ? reinterpret_cast<Device *>(d)->launches : 0;
}

}  // extern "C"
