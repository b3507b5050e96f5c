// Host-side symbolic analysis + first pivoted numeric LU (the one-time step that stays on
// the CPU).  Bit-exact with the reference:
//   min_degree_order   ordering.py:19-59
//   factorize          direct_lu.py:116-294
//   transpose_map      sparsecore.py:321-330 (CSC view, rows ascending per column)
// Compiled with -ffp-contract=off: numpy computes x - (l*xr) with two roundings, and the
// pivot choice depends on those values, so fused multiply-adds would change the pattern.
#include "kkt_internal.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <set>
#include <string>
#include <utility>
#include <vector>

namespace kkt {

thread_local std::string g_last_error;

int set_error(int code, const std::string &msg) {
  g_last_error = msg;
  return code;
}

// ---------------------------------------------------------------------------
// Exact minimum degree on pattern(A + A^T) with explicit clique formation.
// ordering.py:28-59: argmin of degree over alive nodes (smallest index on ties);
// dense tail when degree >= 0.85*(remaining-1) and remaining > 2 -> rest ascending.
// Adjacency is kept as sorted vectors; (degree, index) pairs live in an ordered set
// so the argmin with the smallest-index tie-break is set.begin().
// ---------------------------------------------------------------------------
static const double kDenseTailFraction = 0.85;  // ordering.py:16

void min_degree(int64_t n, const int64_t *rp, const int64_t *ci, std::vector<int64_t> &order) {
  std::vector<std::vector<int32_t>> adj(n);
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
      int64_t j = ci[p];
      if (j != i) {
        adj[i].push_back((int32_t)j);
        adj[j].push_back((int32_t)i);
      }
    }
  }
  for (auto &a : adj) {
    std::sort(a.begin(), a.end());
    a.erase(std::unique(a.begin(), a.end()), a.end());
  }
  std::vector<int64_t> degree(n);
  std::set<std::pair<int64_t, int32_t>> pq;
  for (int64_t i = 0; i < n; ++i) {
    degree[i] = (int64_t)adj[i].size();
    pq.insert({degree[i], (int32_t)i});
  }
  std::vector<char> alive(n, 1);
  order.assign(n, 0);
  std::vector<int32_t> merged;
  for (int64_t step = 0; step < n; ++step) {
    int64_t remaining = n - step;
    int32_t v = pq.begin()->second;
    if (remaining > 2 && (double)degree[v] >= kDenseTailFraction * (double)(remaining - 1)) {
      int64_t s = step;
      for (int64_t i = 0; i < n; ++i)
        if (alive[i]) order[s++] = i;
      return;
    }
    order[step] = v;
    alive[v] = 0;
    pq.erase(pq.begin());
    std::vector<int32_t> nbrs;
    nbrs.swap(adj[v]);  // adj[v] = set()
    for (int32_t u : nbrs) {
      // au.discard(v); au |= nbrs; au.discard(u)
      std::vector<int32_t> &au = adj[u];
      merged.clear();
      merged.reserve(au.size() + nbrs.size());
      size_t a = 0, b = 0;
      while (a < au.size() || b < nbrs.size()) {
        int32_t w;
        if (b >= nbrs.size() || (a < au.size() && au[a] < nbrs[b])) {
          w = au[a++];
        } else if (a >= au.size() || nbrs[b] < au[a]) {
          w = nbrs[b++];
        } else {
          w = au[a++];
          ++b;
        }
        if (w != v && w != u) merged.push_back(w);
      }
      au.swap(merged);
      int64_t nd = (int64_t)au.size();
      if (nd != degree[u]) {
        pq.erase({degree[u], u});
        degree[u] = nd;
        pq.insert({nd, u});
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Left-looking Gilbert-Peierls LU with threshold partial pivoting, recording the replay
// schedule (direct_lu.py:116-294).
// ---------------------------------------------------------------------------
int analyze(int64_t n, const int64_t *rp, const int64_t *ci, const double *av,
            double pivot_tol, Symbolic &S) {
  if (n < 0) return set_error(KKT_ERR_BAD_SHAPE, "factorize requires a square matrix");
  if (!(pivot_tol > 0.0 && pivot_tol <= 1.0))
    return set_error(KKT_ERR_BAD_ARG, "pivot_tol must lie in (0, 1]");
  const int64_t nnz = rp[n];
  S = Symbolic();
  S.n = n;
  S.nnz_a = nnz;
  S.A_row_ptr.assign(rp, rp + n + 1);
  S.A_col_idx.assign(ci, ci + nnz);

  min_degree(n, rp, ci, S.col_perm);

  // transpose_map: CSC with rows ascending per column; vmap = general entry index.
  std::vector<int64_t> cptr(n + 1, 0), cidx(nnz), vmap(nnz);
  for (int64_t p = 0; p < nnz; ++p) cptr[ci[p] + 1]++;
  for (int64_t i = 0; i < n; ++i) cptr[i + 1] += cptr[i];
  {
    std::vector<int64_t> fill(cptr.begin(), cptr.end() - 1);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
        int64_t q = fill[ci[p]]++;
        cidx[q] = i;
        vmap[q] = p;
      }
  }

  std::vector<int64_t> pinv(n, -1), row_perm(n, 0), visited(n, -1);
  std::vector<double> x(n, 0.0);
  std::vector<std::vector<int64_t>> l_rows(n), u_steps(n), solve_orders(n);
  std::vector<std::vector<double>> l_vals(n), u_vals(n);
  std::vector<double> udiag(n, 0.0);

  double max_abs_a = 0.0;
  for (int64_t p = 0; p < nnz; ++p) max_abs_a = std::max(max_abs_a, std::fabs(av[p]));
  double gmax = 0.0;

  std::vector<int64_t> topo, pattern, nonpiv, piv_rows;
  std::vector<std::pair<int64_t, int64_t>> stack;
  for (int64_t j = 0; j < n; ++j) {
    const int64_t c = S.col_perm[j];
    const int64_t s = cptr[c], e = cptr[c + 1];
    if (e == s) {
      char buf[128];
      snprintf(buf, sizeof buf, "structurally singular: column %lld is empty", (long long)c);
      return set_error(KKT_ERR_SINGULAR, buf);
    }
    // Depth-first reach over the graph of the L columns built so far (:169-197).
    topo.clear();
    pattern.clear();
    for (int64_t q = s; q < e; ++q) {
      const int64_t r0 = cidx[q];
      if (visited[r0] == j) continue;
      stack.clear();
      stack.push_back({r0, 0});
      visited[r0] = j;
      while (!stack.empty()) {
        int64_t node = stack.back().first;
        int64_t cix = stack.back().second;
        int64_t k = pinv[node];
        if (k >= 0) {
          const std::vector<int64_t> &children = l_rows[k];
          bool advanced = false;
          while (cix < (int64_t)children.size()) {
            int64_t child = children[cix];
            ++cix;
            if (visited[child] != j) {
              visited[child] = j;
              stack.back().second = cix;
              stack.push_back({child, 0});
              advanced = true;
              break;
            }
          }
          if (advanced) continue;
        }
        stack.pop_back();
        pattern.push_back(node);
        if (k >= 0) topo.push_back(node);
      }
    }
    std::reverse(topo.begin(), topo.end());

    for (int64_t q = s; q < e; ++q) x[cidx[q]] = av[vmap[q]];
    for (int64_t r : topo) {
      const int64_t k = pinv[r];
      const double xr = x[r];
      const std::vector<int64_t> &lr = l_rows[k];
      const std::vector<double> &lv = l_vals[k];
      for (size_t t = 0; t < lr.size(); ++t) {
        double prod = lv[t] * xr;  // separate rounding (no FMA: -ffp-contract=off)
        x[lr[t]] = x[lr[t]] - prod;
      }
    }

    nonpiv.clear();
    for (int64_t r : pattern)
      if (pinv[r] < 0) nonpiv.push_back(r);
    if (nonpiv.empty()) {
      char buf[128];
      snprintf(buf, sizeof buf, "structurally singular: no pivot candidate in column %lld",
               (long long)c);
      return set_error(KKT_ERR_SINGULAR, buf);
    }
    std::sort(nonpiv.begin(), nonpiv.end());
    // amax = max |x[nonpiv]|; argmax = first maximum (np.argmax; NaN wins first).
    double amax = -1.0;
    int64_t iarg = -1;
    bool saw_nan = false;
    for (size_t t = 0; t < nonpiv.size(); ++t) {
      double a = std::fabs(x[nonpiv[t]]);
      if (std::isnan(a)) {
        if (!saw_nan) {
          saw_nan = true;
          iarg = (int64_t)t;
          amax = a;
        }
        continue;
      }
      if (!saw_nan && a > amax) {
        amax = a;
        iarg = (int64_t)t;
      }
    }
    if (amax == 0.0) {
      char buf[160];
      snprintf(buf, sizeof buf,
               "numerically singular: zero pivot column %lld with no admissible swap",
               (long long)c);
      return set_error(KKT_ERR_SINGULAR, buf);
    }
    int64_t ipiv;
    if (pinv[c] < 0 && std::fabs(x[c]) >= pivot_tol * amax)
      ipiv = c;
    else
      ipiv = nonpiv[iarg];
    pinv[ipiv] = j;
    row_perm[j] = ipiv;
    const double ujj = x[ipiv];

    piv_rows.clear();
    for (int64_t r : pattern)
      if (pinv[r] >= 0 && r != ipiv) piv_rows.push_back(r);
    std::vector<std::pair<int64_t, double>> us;
    us.reserve(piv_rows.size());
    double umax = 0.0;
    for (int64_t r : piv_rows) {
      us.push_back({pinv[r], x[r]});
      umax = std::max(umax, std::fabs(x[r]));
    }
    std::sort(us.begin(), us.end(),
              [](const std::pair<int64_t, double> &a, const std::pair<int64_t, double> &b) {
                return a.first < b.first;
              });
    u_steps[j].resize(us.size());
    u_vals[j].resize(us.size());
    for (size_t t = 0; t < us.size(); ++t) {
      u_steps[j][t] = us[t].first;
      u_vals[j][t] = us[t].second;
    }
    udiag[j] = ujj;
    gmax = std::max(gmax, std::max(amax, piv_rows.empty() ? 0.0 : umax));

    std::vector<int64_t> &lr = l_rows[j];
    std::vector<double> &lv = l_vals[j];
    lr.clear();
    lv.clear();
    for (int64_t r : nonpiv)
      if (r != ipiv) {
        lr.push_back(r);
        lv.push_back(x[r] / ujj);
      }
    solve_orders[j].resize(topo.size());
    for (size_t t = 0; t < topo.size(); ++t) solve_orders[j][t] = pinv[topo[t]];
    for (int64_t r : pattern) x[r] = 0.0;
  }

  // Finalize to pivot-position space (:255-285).
  S.row_perm = row_perm;
  S.Lp.assign(n + 1, 0);
  S.Up.assign(n + 1, 0);
  for (int64_t j = 0; j < n; ++j) {
    S.Lp[j + 1] = S.Lp[j] + (int64_t)l_rows[j].size();
    S.Up[j + 1] = S.Up[j] + (int64_t)u_steps[j].size();
  }
  S.Li.resize(S.Lp[n]);
  S.Lx.resize(S.Lp[n]);
  S.Ui.resize(S.Up[n]);
  S.Ux.resize(S.Up[n]);
  std::vector<std::pair<int64_t, double>> tmp;
  for (int64_t j = 0; j < n; ++j) {
    tmp.clear();
    for (size_t t = 0; t < l_rows[j].size(); ++t) tmp.push_back({pinv[l_rows[j][t]], l_vals[j][t]});
    std::sort(tmp.begin(), tmp.end(),
              [](const std::pair<int64_t, double> &a, const std::pair<int64_t, double> &b) {
                return a.first < b.first;
              });
    int64_t base = S.Lp[j];
    for (size_t t = 0; t < tmp.size(); ++t) {
      S.Li[base + t] = tmp[t].first;
      S.Lx[base + t] = tmp[t].second;
    }
    base = S.Up[j];
    for (size_t t = 0; t < u_steps[j].size(); ++t) {
      S.Ui[base + t] = u_steps[j][t];
      S.Ux[base + t] = u_vals[j][t];
    }
  }
  S.Udiag = udiag;
  S.so_ptr.assign(n + 1, 0);
  for (int64_t j = 0; j < n; ++j) S.so_ptr[j + 1] = S.so_ptr[j] + (int64_t)solve_orders[j].size();
  S.so_data.resize(S.so_ptr[n]);
  for (int64_t j = 0; j < n; ++j)
    std::copy(solve_orders[j].begin(), solve_orders[j].end(), S.so_data.begin() + S.so_ptr[j]);
  S.ap_ptr.assign(n + 1, 0);
  for (int64_t j = 0; j < n; ++j) {
    int64_t c = S.col_perm[j];
    S.ap_ptr[j + 1] = S.ap_ptr[j] + (cptr[c + 1] - cptr[c]);
  }
  S.a_src.resize(S.ap_ptr[n]);
  S.a_tgt.resize(S.ap_ptr[n]);
  for (int64_t j = 0; j < n; ++j) {
    int64_t c = S.col_perm[j];
    int64_t base = S.ap_ptr[j];
    for (int64_t q = cptr[c]; q < cptr[c + 1]; ++q) {
      S.a_src[base + (q - cptr[c])] = vmap[q];
      S.a_tgt[base + (q - cptr[c])] = pinv[cidx[q]];
    }
  }
  double maxd = 0.0, mind = 0.0;
  if (n) {
    maxd = std::fabs(udiag[0]);
    mind = maxd;
    for (int64_t j = 1; j < n; ++j) {
      double a = std::fabs(udiag[j]);
      maxd = std::max(maxd, a);
      mind = std::min(mind, a);
    }
  }
  S.diag[0] = maxd;
  S.diag[1] = mind;
  S.diag[2] = 0.0;
  S.diag[3] = max_abs_a > 0 ? gmax / max_abs_a : 0.0;
  compute_schedule_stats(S);
  return KKT_OK;
}

// Level counts of the three DAGs and work figures (reported with every benchmark).
void compute_schedule_stats(Symbolic &S) {
  const int64_t n = S.n;
  std::vector<int32_t> lev(n, 0);
  int64_t max_ref = 0, pairs = 0, max_so = 0;
  for (int64_t j = 0; j < n; ++j) {
    int32_t l = 0;
    for (int64_t p = S.so_ptr[j]; p < S.so_ptr[j + 1]; ++p) {
      int64_t k = S.so_data[p];
      l = std::max(l, lev[k] + 1);
      pairs += S.Lp[k + 1] - S.Lp[k];
    }
    lev[j] = l;
    max_ref = std::max<int64_t>(max_ref, l + 1);
    max_so = std::max<int64_t>(max_so, S.so_ptr[j + 1] - S.so_ptr[j]);
  }
  // L solve (forward): row r depends on column j<r with L(r,j) != 0.
  std::fill(lev.begin(), lev.end(), 0);
  int64_t max_l = 0, max_lcol = 0;
  for (int64_t j = 0; j < n; ++j) {
    max_lcol = std::max<int64_t>(max_lcol, S.Lp[j + 1] - S.Lp[j]);
    for (int64_t p = S.Lp[j]; p < S.Lp[j + 1]; ++p) {
      int64_t r = S.Li[p];
      lev[r] = std::max(lev[r], lev[j] + 1);
    }
    max_l = std::max<int64_t>(max_l, lev[j] + 1);
  }
  // U solve (backward): row r depends on column j>r with U(r,j) != 0.
  std::fill(lev.begin(), lev.end(), 0);
  int64_t max_u = 0, max_ucol = 0;
  for (int64_t j = n - 1; j >= 0; --j) {
    max_ucol = std::max<int64_t>(max_ucol, S.Up[j + 1] - S.Up[j]);
    for (int64_t p = S.Up[j]; p < S.Up[j + 1]; ++p) {
      int64_t r = S.Ui[p];
      lev[r] = std::max(lev[r], lev[j] + 1);
    }
    max_u = std::max<int64_t>(max_u, lev[j] + 1);
  }
  std::vector<int64_t> lrow(n, 0), urow(n, 0);
  for (int64_t p = 0; p < (int64_t)S.Li.size(); ++p) lrow[S.Li[p]]++;
  for (int64_t p = 0; p < (int64_t)S.Ui.size(); ++p) urow[S.Ui[p]]++;
  S.stats[0] = max_ref;
  S.stats[1] = max_l;
  S.stats[2] = max_u;
  S.stats[3] = pairs;
  S.stats[4] = max_so;
  S.stats[5] = max_lcol;
  S.stats[6] = max_ucol;
  S.stats[7] = n ? *std::max_element(lrow.begin(), lrow.end()) : 0;
  S.stats[8] = n ? *std::max_element(urow.begin(), urow.end()) : 0;
}

}  // namespace kkt

// ----------------------------- C ABI ---------------------------------------
extern "C" {

const char *kkt_last_error(void) { return kkt::g_last_error.c_str(); }
int kkt_abi_version(void) { return KKT_ABI_VERSION; }

int kkt_analyze(int64_t n, const int64_t *row_ptr, const int64_t *col_idx, const double *values,
                double pivot_tol, kkt_symbolic **out) {
  if (!out) return kkt::set_error(KKT_ERR_BAD_ARG, "out is NULL");
  *out = nullptr;
  try {
    kkt::Symbolic *S = new kkt::Symbolic();
    int rc = kkt::analyze(n, row_ptr, col_idx, values, pivot_tol, *S);
    if (rc != KKT_OK) {
      delete S;
      return rc;
    }
    *out = reinterpret_cast<kkt_symbolic *>(S);
    return KKT_OK;
  } catch (std::bad_alloc &) {
    return kkt::set_error(KKT_ERR_OOM, "host allocation failed in kkt_analyze");
  }
}

int kkt_min_degree_order(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                         int64_t *perm_out) {
  try {
    std::vector<int64_t> order;
    kkt::min_degree(n, row_ptr, col_idx, order);
    std::copy(order.begin(), order.end(), perm_out);
    return KKT_OK;
  } catch (std::bad_alloc &) {
    return kkt::set_error(KKT_ERR_OOM, "host allocation failed in min_degree_order");
  }
}

void kkt_symbolic_free(kkt_symbolic *s) { delete reinterpret_cast<kkt::Symbolic *>(s); }

int kkt_symbolic_sizes(const kkt_symbolic *s, int64_t sizes[KKT_SZ_COUNT]) {
  const kkt::Symbolic *S = reinterpret_cast<const kkt::Symbolic *>(s);
  if (!S) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL symbolic");
  sizes[KKT_SZ_N] = S->n;
  sizes[KKT_SZ_NNZ_A] = S->nnz_a;
  sizes[KKT_SZ_NNZ_L] = (int64_t)S->Li.size();
  sizes[KKT_SZ_NNZ_U] = (int64_t)S->Ui.size();
  sizes[KKT_SZ_NSO] = (int64_t)S->so_data.size();
  sizes[KKT_SZ_NAP] = (int64_t)S->a_src.size();
  return KKT_OK;
}

#define KKT_COPY(dst, vec) \
  if (dst) std::copy(S->vec.begin(), S->vec.end(), dst)

int kkt_symbolic_export(const kkt_symbolic *s, int64_t *row_perm, int64_t *col_perm, int64_t *Lp,
                        int64_t *Li, double *Lx, int64_t *Up, int64_t *Ui, double *Ux,
                        double *Udiag, int64_t *so_ptr, int64_t *so_data, int64_t *ap_ptr,
                        int64_t *a_src, int64_t *a_tgt) {
  const kkt::Symbolic *S = reinterpret_cast<const kkt::Symbolic *>(s);
  if (!S) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL symbolic");
  KKT_COPY(row_perm, row_perm);
  KKT_COPY(col_perm, col_perm);
  KKT_COPY(Lp, Lp);
  KKT_COPY(Li, Li);
  KKT_COPY(Lx, Lx);
  KKT_COPY(Up, Up);
  KKT_COPY(Ui, Ui);
  KKT_COPY(Ux, Ux);
  KKT_COPY(Udiag, Udiag);
  KKT_COPY(so_ptr, so_ptr);
  KKT_COPY(so_data, so_data);
  KKT_COPY(ap_ptr, ap_ptr);
  KKT_COPY(a_src, a_src);
  KKT_COPY(a_tgt, a_tgt);
  return KKT_OK;
}

int kkt_symbolic_diag(const kkt_symbolic *s, double diag[4]) {
  const kkt::Symbolic *S = reinterpret_cast<const kkt::Symbolic *>(s);
  if (!S) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL symbolic");
  for (int i = 0; i < 4; ++i) diag[i] = S->diag[i];
  return KKT_OK;
}

int kkt_symbolic_stats(const kkt_symbolic *s, int64_t stats[9]) {
  const kkt::Symbolic *S = reinterpret_cast<const kkt::Symbolic *>(s);
  if (!S) return kkt::set_error(KKT_ERR_BAD_ARG, "NULL symbolic");
  for (int i = 0; i < 9; ++i) stats[i] = S->stats[i];
  return KKT_OK;
}

}  // extern "C"
