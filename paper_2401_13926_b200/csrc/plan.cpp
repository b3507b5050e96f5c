// Host-side construction of the device execution plan from the analysis (one-time, part of
// kkt_dev_create).  Everything here is integer bookkeeping over the frozen pattern:
//   * refactor: column dispatch order (by DAG level), per-column workspace slots, the
//     relative slot of every update pair (uint16), A-scatter slots, CSC->CSR value maps;
//   * trisolves: CSR of L (ascending columns) and U (descending columns, so the reference's
//     descending-j accumulation order is a forward walk), row dispatch order by level;
//   * SpMV: split point of each general row so the reference's symmetric-lower bincount
//     order (sparsecore.py:296-302) is reproduced.
#include "plan.h"

#include <algorithm>
#include <cstdlib>
#include <numeric>

namespace kkt {

static std::vector<int32_t> order_by_level(const std::vector<int32_t> &lev) {
  const int64_t n = (int64_t)lev.size();
  int32_t nl = 0;
  for (int32_t l : lev) nl = std::max(nl, l + 1);
  std::vector<int64_t> cnt(nl + 1, 0);
  for (int32_t l : lev) cnt[l + 1]++;
  for (int32_t l = 0; l < nl; ++l) cnt[l + 1] += cnt[l];
  std::vector<int32_t> out(n);
  for (int64_t i = 0; i < n; ++i) out[cnt[lev[i]]++] = (int32_t)i;  // stable: ascending within level
  return out;
}

// L: blocks ascend from p (rows r >= block end receive the off-diagonal updates);
// U: blocks descend from n (rows p <= r < block start receive them).  CSR rows are column-
// ascending for L and column-descending for U, so each row's entries inside a block are one
// contiguous run, already in the reference's per-row order.
static void build_sweep(const HostPlan &P, bool upper, HostSweep &H) {
  const int32_t n = P.n, p = upper ? P.pU : P.pL, T = n - p;
  const std::vector<int32_t> &rp = upper ? P.Urp : P.Lrp, &ci = upper ? P.Uci : P.Lci;
  H = HostSweep();
  H.nblk = (T + 31) / 32;
  H.dptr.assign(1, 0);
  H.bptr.assign(1, 0);
  H.dmask.assign((size_t)H.nblk * 32, 0u);
  for (int32_t c = 0; c < H.nblk; ++c) {
    int32_t lo, w;
    if (!upper) {
      lo = p + 32 * c;
      w = std::min(32, n - lo);
    } else {
      const int32_t hi = n - 32 * c;
      lo = std::max(p, hi - 32);
      w = hi - lo;
    }
    auto run = [&](int32_t r, int32_t &beg, int32_t &cnt) {  // entries of row r in [lo, lo+w)
      beg = rp[r];
      while (beg < rp[r + 1] && !(ci[beg] >= lo && ci[beg] < lo + w)) ++beg;
      cnt = 0;
      while (beg + cnt < rp[r + 1] && ci[beg + cnt] >= lo && ci[beg + cnt] < lo + w) ++cnt;
    };
    for (int32_t i = 0; i < w; ++i) {
      int32_t beg, cnt;
      run(lo + i, beg, cnt);
      for (int32_t k = 0; k < cnt; ++k) {
        const int32_t t = ci[beg + k] - lo;
        H.dsrc.push_back(beg + k);
        H.ddst.push_back((uint16_t)(i * 32 + t));
        H.dmask[(size_t)c * 32 + i] |= 1u << t;
      }
    }
    H.dptr.push_back((int32_t)H.dsrc.size());
    const int32_t r0 = upper ? p : lo + w, r1 = upper ? lo : n;
    int32_t staged = 0;
    for (int32_t r = r0; r < r1; ++r) {
      int32_t beg, cnt;
      run(r, beg, cnt);
      if (cnt) {
        H.brow.push_back(r);
        H.bbeg.push_back(beg);
        H.bcnt.push_back(cnt);
        H.bofs.push_back(staged);  // position of the run in the block's shared-memory stage
        staged += cnt;
      }
    }
    H.max_stage = std::max(H.max_stage, staged);
    H.bptr.push_back((int32_t)H.brow.size());
  }
}

// Single-system grid phase as chain tasks (trisolve.cu k_trsv_chain).  A chain is a run of up
// to 32 consecutive grid rows, each depending on its predecessor in the solve order (L: row
// r-1 -> r, U: r+1 -> r).  One warp solves it row by row, lane i holding row i, so a link of
// the chain costs a shuffle instead of an L2 publish/poll round trip (at 10k the grid phases
// have 196 levels each, but only 28 once such runs are contracted).  A chain row's entries
// split into external columns (outside the chain) and internal ones, and the external ones
// come first in the row's update order (L ascending columns < r0, U descending columns > r0),
// so their sum is an independent "partial" task (warp per row, published into cpart) that the
// chain warp waits for.  Tasks are sorted by a modelled start time (HOP per L2 hand-off, LINK
// per chain row) — every dependency finishes strictly before a task's modelled start, so the
// order is topological and the persistent grid cannot deadlock.
static void build_chains(HostPlan &P, bool upper) {
  const double HOP = 1.5, LINK = 0.15;
  const int32_t p = upper ? P.pU : P.pL;
  const std::vector<int32_t> &rp = upper ? P.Urp : P.Lrp, &ci = upper ? P.Uci : P.Lci;
  std::vector<int32_t> &task = upper ? P.Uc_task : P.Lc_task, &aux = upper ? P.Uc_aux : P.Lc_aux,
                       &split = upper ? P.Uc_split : P.Lc_split;
  task.clear();
  aux.clear();
  split.assign(std::max<int32_t>(p, 1), 0);
  if (p <= 0 || P.n >= (1 << 26)) return;
  std::vector<char> grid(p, 1);  // L: the leading levels run row-parallel before the grid
  if (!upper)
    for (int32_t i = 0; i < P.L_sync_ptr.back(); ++i) grid[P.L_grid_order[i]] = 0;
  auto gbeg = [&](int32_t r) { return upper ? P.Ugrid_split[r] : rp[r]; };
  // chain heads and lengths, walking the solve order
  std::vector<int32_t> head(p, -1), len(p, 0);
  for (int32_t s = 0; s < p; ++s) {
    const int32_t r = upper ? p - 1 - s : s;
    if (!grid[r]) continue;
    const int32_t prev = upper ? r + 1 : r - 1;
    const bool link = prev >= 0 && prev < p && grid[prev] && rp[r + 1] > gbeg(r) &&
                      ci[rp[r + 1] - 1] == prev && len[head[prev]] < 32;
    head[r] = link ? head[prev] : r;
    len[head[r]]++;
  }
  struct T {
    double t;
    int32_t code, aux;
  };
  std::vector<T> tl;
  tl.reserve(p);
  std::vector<double> fin(p, 0.0);
  // latest-finishing grid dependency among the entries [q0, q1) of a row
  auto latest = [&](int32_t q0, int32_t q1, double *tmax) {
    int32_t best = -1;
    double bt = -1.0;
    for (int32_t q = q0; q < q1; ++q) {
      const int32_t c = ci[q];
      if (c >= p || !grid[c]) continue;
      if (fin[c] > bt) {
        bt = fin[c];
        best = c;
      }
    }
    *tmax = std::max(bt, 0.0);
    return best;
  };
  for (int32_t s = 0; s < p; ++s) {
    const int32_t h = upper ? p - 1 - s : s;
    if (!grid[h] || head[h] != h) continue;
    const int32_t m = len[h];
    if (m == 1) {
      double t;
      const int32_t cr = latest(gbeg(h), rp[h + 1], &t);
      fin[h] = t + HOP;
      tl.push_back({t + HOP, h, cr});
      continue;
    }
    double start = 0.0;
    uint32_t mask = 0;
    for (int32_t i = 0; i < m; ++i) {
      const int32_t r = upper ? h - i : h + i;
      int32_t q = gbeg(r);
      while (q < rp[r + 1] && (upper ? ci[q] > h : ci[q] < h)) ++q;
      split[r] = q;
      if (q > gbeg(r)) {  // external entries: a partial task
        double t;
        const int32_t cr = latest(gbeg(r), q, &t);
        tl.push_back({t + HOP, -(r + 1), cr});
        mask |= 1u << i;
        start = std::max(start, t + HOP);
      }
    }
    start += HOP;
    tl.push_back({start, h | ((m - 1) << 26), (int32_t)mask});
    for (int32_t i = 0; i < m; ++i) fin[upper ? h - i : h + i] = start + LINK * (i + 1);
  }
  std::stable_sort(tl.begin(), tl.end(), [](const T &a, const T &b) { return a.t < b.t; });
  task.resize(tl.size());
  aux.resize(tl.size());
  for (size_t i = 0; i < tl.size(); ++i) {
    task[i] = tl[i].code;
    aux[i] = tl[i].aux;
  }
}

// Invariants of the chain task lists (kkt_plan_check; host only).  out: {tasks L, tasks U,
// chains, chain rows, longest chain, order violations, coverage violations, 0}.  An order
// violation is a task that reads a value (a y of the grid phase, or a chain row's prefix sum)
// produced by a task at the same or a later position — the persistent grid is deadlock-free
// exactly when there are none, since every warp takes its tasks in list order.
void check_chains(const HostPlan &P, int64_t out[8]) {
  for (int i = 0; i < 8; ++i) out[i] = 0;
  for (int up = 0; up < 2; ++up) {
    const bool upper = up != 0;
    const int32_t p = upper ? P.pU : P.pL;
    const std::vector<int32_t> &rp = upper ? P.Urp : P.Lrp, &ci = upper ? P.Uci : P.Lci;
    const std::vector<int32_t> &task = upper ? P.Uc_task : P.Lc_task, &aux = upper ? P.Uc_aux : P.Lc_aux,
                               &split = upper ? P.Uc_split : P.Lc_split;
    out[up] = (int64_t)task.size();
    if (p <= 0) continue;
    std::vector<char> grid(p, 1);
    if (!upper)
      for (int32_t i = 0; i < P.L_sync_ptr.back(); ++i) grid[P.L_grid_order[i]] = 0;
    auto gbeg = [&](int32_t r) { return upper ? P.Ugrid_split[r] : rp[r]; };
    std::vector<int64_t> prod(p, -1), pre(p, -1);  // task publishing y[r] / r's prefix sum
    for (size_t t = 0; t < task.size(); ++t) {
      const int32_t c = task[t];
      auto own = [&](int32_t r, std::vector<int64_t> &v) {
        if (r < 0 || r >= p || !grid[r] || v[r] >= 0) ++out[6];
        else v[r] = (int64_t)t;
      };
      if (c < 0) own(-c - 1, pre);
      else if ((c >> 26) == 0) own(c, prod);
      else {
        const int32_t h = c & ((1 << 26) - 1), m = (c >> 26) + 1;
        ++out[2];
        out[3] += m;
        out[4] = std::max<int64_t>(out[4], m);
        for (int32_t i = 0; i < m; ++i) own(upper ? h - i : h + i, prod);
      }
    }
    for (int32_t r = 0; r < p; ++r)
      if (grid[r] && prod[r] < 0) ++out[6];  // a grid row nobody publishes
    auto before = [&](int32_t col, int64_t t) {  // y[col] is published before task t
      if (col >= p || !grid[col]) return true;    // head columns / row-parallel levels: earlier launches
      return prod[col] >= 0 && prod[col] < t;
    };
    for (size_t t = 0; t < task.size(); ++t) {
      const int32_t c = task[t];
      if (c < 0 || (c >> 26) == 0) {
        const int32_t r = c < 0 ? -c - 1 : c;
        if (r < 0 || r >= p) continue;
        const int32_t end = c < 0 ? split[r] : rp[r + 1];
        for (int32_t q = gbeg(r); q < end; ++q) out[5] += !before(ci[q], (int64_t)t);
        continue;
      }
      const int32_t h = c & ((1 << 26) - 1), m = (c >> 26) + 1;
      const uint32_t mask = (uint32_t)aux[t];
      for (int32_t i = 0; i < m; ++i) {
        const int32_t r = upper ? h - i : h + i;
        const bool ext = split[r] > gbeg(r);
        if (ext != (((mask >> i) & 1u) != 0) || (ext && !(pre[r] >= 0 && pre[r] < (int64_t)t))) ++out[5];
        for (int32_t q = split[r]; q < rp[r + 1]; ++q) {  // internal: earlier rows of this chain
          const int32_t col = ci[q];
          const bool inside = upper ? (col > r && col <= h) : (col < r && col >= h);
          out[6] += !inside;
        }
      }
    }
  }
}

int build_plan(const Symbolic &S, const int64_t *A_rp, const int64_t *A_ci, int64_t in_nnz,
               const int64_t *gen_src, HostPlan &P) {
  const int64_t n = S.n;
  if (n >= (int64_t)INT32_MAX / 2) return set_error(KKT_ERR_BAD_SHAPE, "n too large for int32 plan");
  P = HostPlan();
  P.n = (int32_t)n;
  const int64_t nnz = S.nnz_a;
  for (int64_t i = 0; i <= n; ++i)
    if (A_rp[i] != S.A_row_ptr[i])
      return set_error(KKT_ERR_PATTERN_MISMATCH, "operator pattern differs from the analysed one");
  for (int64_t p = 0; p < nnz; ++p)
    if (A_ci[p] != S.A_col_idx[p])
      return set_error(KKT_ERR_PATTERN_MISMATCH, "operator pattern differs from the analysed one");
  P.nnz_a = nnz;
  P.in_nnz = in_nnz;
  P.A_rp.assign(A_rp, A_rp + n + 1);
  P.A_ci.assign(A_ci, A_ci + nnz);
  P.gen_src.assign(nnz, 0);
  P.has_lower = gen_src != nullptr && in_nnz > 0;
  if (P.has_lower) {
    for (int64_t e = 0; e < nnz; ++e) {
      if (gen_src[e] < 0 || gen_src[e] >= in_nnz)
        return set_error(KKT_ERR_BAD_SHAPE, "gen_src index out of range");
      P.gen_src[e] = gen_src[e];
    }
  } else {
    P.in_nnz = 0;
  }
  // SpMV split: first entry with col > row (symmetric-lower operators sum the halves apart).
  P.A_split.resize(n);
  for (int64_t i = 0; i < n; ++i) {
    int64_t p = A_rp[i];
    while (p < A_rp[i + 1] && A_ci[p] <= i) ++p;
    P.A_split[i] = p;
  }

  // ---------------- refactor ----------------
  const int64_t nL = (int64_t)S.Li.size(), nU = (int64_t)S.Ui.size();
  P.Lp.assign(S.Lp.begin(), S.Lp.end());
  P.Up.assign(S.Up.begin(), S.Up.end());
  P.row_perm.assign(S.row_perm.begin(), S.row_perm.end());
  P.col_perm.assign(S.col_perm.begin(), S.col_perm.end());
  P.nnz_L = nL;
  P.nnz_U = nU;
  // column workspace = U rows (ascending), the diagonal, L rows (ascending): sorted positions
  std::vector<int32_t> pos2slot(n, -1);
  P.so_ptr.assign(S.so_ptr.begin(), S.so_ptr.end());
  const int64_t nso = (int64_t)S.so_data.size();
  P.so_data.resize(nso);
  P.so_slot.resize(nso);
  P.upd_ptr.resize(nso + 1);
  int64_t pairs = 0;
  for (int64_t t = 0; t < nso; ++t) {
    int64_t k = S.so_data[t];
    pairs += S.Lp[k + 1] - S.Lp[k];
  }
  if (pairs >= (int64_t)INT32_MAX) return set_error(KKT_ERR_BAD_SHAPE, "too many update pairs");
  P.upd_slot.resize(pairs);
  P.ap_ptr.assign(S.ap_ptr.begin(), S.ap_ptr.end());
  P.a_src.resize(S.a_src.size());
  P.a_slot.resize(S.a_src.size());
  int32_t maxpat = 1;
  int64_t u = 0;
  std::vector<int32_t> lev(n, 0);
  for (int64_t j = 0; j < n; ++j) {
    const int64_t nu = S.Up[j + 1] - S.Up[j], nl = S.Lp[j + 1] - S.Lp[j];
    const int64_t np = nu + 1 + nl;
    if (np > 65535) return set_error(KKT_ERR_BAD_SHAPE, "column pattern exceeds 65535 slots");
    maxpat = std::max<int32_t>(maxpat, (int32_t)np);
    for (int64_t s = 0; s < nu; ++s) pos2slot[S.Ui[S.Up[j] + s]] = (int32_t)s;
    pos2slot[j] = (int32_t)nu;
    for (int64_t s = 0; s < nl; ++s) pos2slot[S.Li[S.Lp[j] + s]] = (int32_t)(nu + 1 + s);
    int32_t l = 0;
    for (int64_t t = S.so_ptr[j]; t < S.so_ptr[j + 1]; ++t) {
      const int64_t k = S.so_data[t];
      l = std::max(l, lev[k] + 1);
      P.so_data[t] = (int32_t)k;
      P.so_slot[t] = (uint16_t)pos2slot[k];
      P.upd_ptr[t] = (int32_t)u;
      for (int64_t p = S.Lp[k]; p < S.Lp[k + 1]; ++p) {
        int32_t s = pos2slot[S.Li[p]];
        if (s < 0) return set_error(KKT_ERR_BAD_SHAPE, "replay schedule leaves column pattern");
        P.upd_slot[u++] = (uint16_t)s;
      }
    }
    lev[j] = l;
    for (int64_t q = S.ap_ptr[j]; q < S.ap_ptr[j + 1]; ++q) {
      P.a_src[q] = (int32_t)S.a_src[q];
      int32_t s = pos2slot[S.a_tgt[q]];
      if (s < 0) return set_error(KKT_ERR_BAD_SHAPE, "A entry outside column pattern");
      P.a_slot[q] = (uint16_t)s;
    }
    for (int64_t s = 0; s < nu; ++s) pos2slot[S.Ui[S.Up[j] + s]] = -1;
    pos2slot[j] = -1;
    for (int64_t s = 0; s < nl; ++s) pos2slot[S.Li[S.Lp[j] + s]] = -1;
  }
  P.upd_ptr[nso] = (int32_t)u;
  P.so_meta.assign(4 * nso, 0);
  P.upd_lidx.resize(pairs);
  for (int64_t t = 0; t < nso; ++t) {
    const int64_t k = S.so_data[t];
    P.so_meta[4 * t + 0] = P.so_slot[t];
    P.so_meta[4 * t + 1] = (int32_t)(S.Lp[k + 1] - S.Lp[k]);
    P.so_meta[4 * t + 2] = P.upd_ptr[t];
    P.so_meta[4 * t + 3] = (int32_t)S.Lp[k];
    for (int64_t e = 0; e < S.Lp[k + 1] - S.Lp[k]; ++e) P.upd_lidx[P.upd_ptr[t] + e] = (int32_t)(S.Lp[k] + e);
  }
  P.maxpat = maxpat;
  P.col_order = order_by_level(lev);
  P.refactor_levels = 0;
  for (int32_t l : lev) P.refactor_levels = std::max(P.refactor_levels, l + 1);
  {
    // leading levels that are wide (>= 2048 columns) with small patterns (<= 64 slots):
    // thread-per-column launches instead of one warp per column
    std::vector<int64_t> cnt(P.refactor_levels + 1, 0), mp(P.refactor_levels + 1, 0);
    for (int64_t j = 0; j < n; ++j) {
      cnt[lev[j]]++;
      mp[lev[j]] = std::max<int64_t>(mp[lev[j]], S.Up[j + 1] - S.Up[j] + 1 + S.Lp[j + 1] - S.Lp[j]);
    }
    P.small_lev_ptr.assign(1, 0);
    int32_t l = 0;
    int cap = 2;  // KKT_SMALL_LEVELS (<= 8; 4/6/8 measured slower at 10k, batched and single)
    if (const char *e = std::getenv("KKT_SMALL_LEVELS")) cap = std::max(0, std::min(8, std::atoi(e)));
    while (l < P.refactor_levels && l < cap && cnt[l] >= 2048 && mp[l] <= 64) {
      P.small_lev_ptr.push_back(P.small_lev_ptr.back() + (int32_t)cnt[l]);
      ++l;
    }
    P.n_small_levels = l;
  }

  // ---------------- trisolves: CSR of L (ascending cols) and U (descending cols) -------
  P.Lrp.assign(n + 1, 0);
  P.Urp.assign(n + 1, 0);
  for (int64_t p = 0; p < nL; ++p) P.Lrp[S.Li[p] + 1]++;
  for (int64_t p = 0; p < nU; ++p) P.Urp[S.Ui[p] + 1]++;
  for (int64_t i = 0; i < n; ++i) {
    P.Lrp[i + 1] += P.Lrp[i];
    P.Urp[i + 1] += P.Urp[i];
  }
  P.Lci.resize(nL);
  P.Lmap.resize(nL);
  P.Uci.resize(nU);
  P.Umap.resize(nU);
  {
    std::vector<int32_t> fill(P.Lrp.begin(), P.Lrp.end() - 1);
    for (int64_t j = 0; j < n; ++j)  // ascending j => ascending columns per row
      for (int64_t p = S.Lp[j]; p < S.Lp[j + 1]; ++p) {
        int32_t q = fill[S.Li[p]]++;
        P.Lci[q] = (int32_t)j;
        P.Lmap[p] = q;
      }
    std::vector<int32_t> ufill(P.Urp.begin(), P.Urp.end() - 1);
    for (int64_t j = n - 1; j >= 0; --j)  // descending j => descending columns per row
      for (int64_t p = S.Up[j]; p < S.Up[j + 1]; ++p) {
        int32_t q = ufill[S.Ui[p]]++;
        P.Uci[q] = (int32_t)j;
        P.Umap[p] = q;
      }
  }
  // levels: L row r after every column j<r it references; U row r after every j>r.
  std::vector<int32_t> levL(n, 0), levU(n, 0);
  for (int64_t r = 0; r < n; ++r) {
    int32_t l = 0;
    for (int32_t p = P.Lrp[r]; p < P.Lrp[r + 1]; ++p) l = std::max(l, levL[P.Lci[p]] + 1);
    levL[r] = l;
  }
  for (int64_t r = n - 1; r >= 0; --r) {
    int32_t l = 0;
    for (int32_t p = P.Urp[r]; p < P.Urp[r + 1]; ++p) l = std::max(l, levU[P.Uci[p]] + 1);
    levU[r] = l;
  }
  P.L_levels = 0;
  P.U_levels = 0;
  for (int64_t i = 0; i < n; ++i) {
    P.L_levels = std::max(P.L_levels, levL[i] + 1);
    P.U_levels = std::max(P.U_levels, levU[i] + 1);
  }
  // ---- phase split ----
  {
    const int TL = choose_tail(P, false), TU = choose_tail(P, true);
    P.pL = (int32_t)(n - TL);
    P.pU = (int32_t)(n - TU);
    // L grid phase: the rows < pL.  Every tail row's leading entries (columns < pL) are
    // summed by a separate row-parallel launch after it (nothing in the grid waits on them),
    // whose result seeds the sweep.
    std::vector<int32_t> lg(levL.begin(), levL.begin() + P.pL);
    P.Ltail_split.assign(n - P.pL, 0);
    for (int64_t r = P.pL; r < n; ++r) {
      int32_t q = P.Lrp[r];
      while (q < P.Lrp[r + 1] && P.Lci[q] < P.pL) ++q;
      P.Ltail_split[r - P.pL] = q;
    }
    P.L_grid_order = order_by_level(lg);
    P.L_grid_levels = 0;
    for (int32_t l : lg) P.L_grid_levels = std::max(P.L_grid_levels, l + 1);
    // wide leading levels (>= 4096 rows, at most 4) run level-synchronously, row-parallel
    {
      std::vector<int64_t> cnt(P.L_grid_levels + 1, 0);
      for (int32_t l : lg) cnt[l]++;
      P.L_sync_ptr.assign(1, 0);
      for (int32_t l = 0; l < P.L_grid_levels && l < 4 && cnt[l] >= 4096; ++l)
        P.L_sync_ptr.push_back(P.L_sync_ptr.back() + (int32_t)cnt[l]);
    }
    std::vector<int32_t> lt(levL.begin() + P.pL, levL.end());
    P.L_tail_order = order_by_level(lt);
    for (auto &v : P.L_tail_order) v += P.pL;
    // U: head rows [pU, n) keep their levels; grid rows' levels ignore head dependencies
    std::vector<int32_t> uh(levU.begin() + P.pU, levU.end());
    P.U_head_order = order_by_level(uh);
    for (auto &v : P.U_head_order) v += P.pU;
    std::vector<int32_t> lu(P.pU, 0);
    for (int64_t r = P.pU - 1; r >= 0; --r) {
      int32_t l = 0;
      for (int32_t q = P.Urp[r]; q < P.Urp[r + 1]; ++q)
        if (P.Uci[q] < P.pU) l = std::max(l, lu[P.Uci[q]] + 1);
      lu[r] = l;
    }
    P.U_grid_order = order_by_level(lu);
    // the grid rows' head-column prefix (final before the grid phase): summed by a separate
    // row-parallel launch into yL, so the grid kernel starts each row at Ugrid_split
    P.Ugrid_split.assign(P.pU, 0);
    P.U_part_rows.clear();
    for (int64_t r = 0; r < P.pU; ++r) {
      int32_t q = P.Urp[r];
      while (q < P.Urp[r + 1] && P.Uci[q] >= P.pU) ++q;
      P.Ugrid_split[r] = q;
      if (q > P.Urp[r]) P.U_part_rows.push_back((int32_t)r);
    }
    // level boundaries of both grid orders (the batched level-synchronous kernel)
    auto lev_ptr = [](const std::vector<int32_t> &lev, std::vector<int32_t> &ptr) {
      int32_t nl = 0;
      for (int32_t l : lev) nl = std::max(nl, l + 1);
      ptr.assign(nl + 1, 0);
      for (int32_t l : lev) ptr[l + 1]++;
      for (int32_t l = 0; l < nl; ++l) ptr[l + 1] += ptr[l];
    };
    lev_ptr(lg, P.L_glev_ptr);
    lev_ptr(lu, P.U_glev_ptr);
    P.U_grid_levels = 0;
    for (int32_t l : lu) P.U_grid_levels = std::max(P.U_grid_levels, l + 1);
    // critical dependency: highest level, ties -> the most recently finished column
    P.L_crit.assign(P.L_grid_order.size(), -1);
    for (size_t i = 0; i < P.L_grid_order.size(); ++i) {
      const int32_t r = P.L_grid_order[i];
      int32_t best = -1, bl = -1;
      for (int32_t q = P.Lrp[r]; q < P.Lrp[r + 1]; ++q) {
        const int32_t c = P.Lci[q];
        if (levL[c] > bl || (levL[c] == bl && c > best)) {
          bl = levL[c];
          best = c;
        }
      }
      P.L_crit[i] = best;
    }
    P.U_crit.assign(P.U_grid_order.size(), -1);
    for (size_t i = 0; i < P.U_grid_order.size(); ++i) {
      const int32_t r = P.U_grid_order[i];
      int32_t best = -1, bl = -1;
      for (int32_t q = P.Urp[r]; q < P.Urp[r + 1]; ++q) {
        const int32_t c = P.Uci[q];
        if (c >= P.pU) continue;  // head columns are final before the grid phase starts
        if (lu[c] > bl || (lu[c] == bl && c < best)) {
          bl = lu[c];
          best = c;
        }
      }
      P.U_crit[i] = best;
    }
    P.Uhead_off.assign(n - P.pU, 0);
    for (int64_t j = P.pU; j < n; ++j) {
      int64_t q = S.Up[j];
      while (q < S.Up[j + 1] && S.Ui[q] < P.pU) ++q;
      P.Uhead_off[j - P.pU] = (int32_t)(q - S.Up[j]);
    }
    for (int64_t j = P.pL; j < n; ++j)
      P.sweep_maxL = std::max<int32_t>(P.sweep_maxL, (int32_t)(S.Lp[j + 1] - S.Lp[j]));
    for (int64_t j = P.pU; j < n; ++j)
      P.sweep_maxU = std::max<int32_t>(P.sweep_maxU,
                                       (int32_t)(S.Up[j + 1] - S.Up[j] - P.Uhead_off[j - P.pU]));
    P.Li32.assign(S.Li.begin(), S.Li.end());
    P.Ui32.assign(S.Ui.begin(), S.Ui.end());
    build_sweep(P, false, P.swL);
    build_sweep(P, true, P.swU);
    build_chains(P, false);
    build_chains(P, true);
  }
  P.Lx0.assign(S.Lx.begin(), S.Lx.end());
  P.Ux0.assign(S.Ux.begin(), S.Ux.end());
  P.Udiag0.assign(S.Udiag.begin(), S.Udiag.end());
  return KKT_OK;
}

// Cost model for the sweep-phase size T (the last T positions): each grid-phase level costs
// ~GRID_HOP_US (an L2 round trip on the dependency chain), each sweep column ~SWEEP_COL_US
// (the blocked sweep's per-column chain) plus ~SWEEP_NNZ_US per block entry of throughput.
// SWEEP_COL_US refitted after the grid phases got faster (batched without the up-front wait,
// single-system chain tasks): measured optimum T = 256..768 at 10k (single 0.87-0.89 ms vs
// 0.98 at the old choice 1,536; batch of 64 1.54 vs 1.72 ms) and 512 at 70k (2.83 vs 3.25).
int choose_tail(const HostPlan &P, bool upper) {
  const char *env = std::getenv(upper ? "KKT_HEAD_ROWS" : "KKT_TAIL_ROWS");
  const int n = P.n;
  if (env) return std::max(0, std::min(n, std::min(atoi(env), KKT_CTA_PHASE_MAX_ROWS)));
  const double GRID_HOP_US = 1.0, SWEEP_COL_US = 0.2, SWEEP_NNZ_US = 0.0003;
  const std::vector<int32_t> &rp = upper ? P.Urp : P.Lrp;
  const std::vector<int32_t> &ci = upper ? P.Uci : P.Lci;
  double best = 1e30;
  int bestT = 0;
  for (int T : {0, 32, 64, 128, 256, 512, 768, 1024, 1536, 2048, 3072, 4096}) {
    if (T > n || T > KKT_CTA_PHASE_MAX_ROWS) break;
    const int p = n - T;
    // levels of the grid part and of the CTA part
    std::vector<int32_t> lev(n, 0);
    int32_t gl = 0, tl = 0;
    if (!upper) {
      for (int r = 0; r < n; ++r) {
        int32_t l = 0;
        for (int32_t q = rp[r]; q < rp[r + 1]; ++q)
          if ((r < p) == (ci[q] < p)) l = std::max(l, lev[ci[q]] + 1);
        lev[r] = l;
        if (r < p) gl = std::max(gl, l + 1); else tl = std::max(tl, l + 1);
      }
    } else {
      for (int r = n - 1; r >= 0; --r) {
        int32_t l = 0;
        for (int32_t q = rp[r]; q < rp[r + 1]; ++q)
          if ((r < p) == (ci[q] < p)) l = std::max(l, lev[ci[q]] + 1);
        lev[r] = l;
        if (r < p) gl = std::max(gl, l + 1); else tl = std::max(tl, l + 1);
      }
    }
    const int64_t tnnz = T ? (int64_t)(rp[n] - rp[p]) : 0;
    (void)tl;
    const double cost = GRID_HOP_US * gl + SWEEP_COL_US * T + SWEEP_NNZ_US * (double)tnnz;
    if (cost < best) {
      best = cost;
      bestT = T;
    }
  }
  return bestT;
}

}  // namespace kkt
