/*
 * kkt_oracle.c — CPU ORACLE (test infrastructure, NOT product code).
 *
 * A plain-C restatement of the reference hot path (kktsolve, pkg/src/kktsolve/...), used
 * only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs as the checker and the CPU timing baseline.  Never linked into libkktb200.so.
 *
 * Pinned against the tests/golden fixtures (outputs of the reference itself, produced by
 * tests/golden/make_golden.py): tests/test_oracle.py.
 *
 * Every floating-point statement keeps numpy's rounding sequence (compile with
 * -ffp-contract=off): products and differences round separately.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* sparsecore.inf_norm (sparsecore.py:333-343): row sums of |a| in entry order (bincount);
 * symmetric-lower storage adds the mirrored strict entries in a second bincount. */
double oracle_inf_norm(int64_t n, const int64_t *rp, const int64_t *ci, const double *v,
                       int sym_lower) {
  double *s1 = calloc(n ? n : 1, sizeof(double)), *s2 = calloc(n ? n : 1, sizeof(double));
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
      s1[i] = s1[i] + fabs(v[p]);
      if (sym_lower && ci[p] != i) s2[ci[p]] = s2[ci[p]] + fabs(v[p]);
    }
  double m = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double t = sym_lower ? s1[i] + s2[i] : s1[i];
    if (i == 0 || t > m) m = t;
  }
  free(s1);
  free(s2);
  return n ? m : 0.0;
}

/* sparsecore.spmv (sparsecore.py:284-305): y = bincount(rows, v*x[col]) (+ mirrored). */
void oracle_spmv(int64_t n, const int64_t *rp, const int64_t *ci, const double *v, int sym_lower,
                 const double *x, double *y) {
  double *t = sym_lower ? calloc(n ? n : 1, sizeof(double)) : NULL;
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
      double prod = v[p] * x[ci[p]];
      acc = acc + prod;
      if (sym_lower && ci[p] != i) {
        double q = v[p] * x[i];
        t[ci[p]] = t[ci[p]] + q;
      }
    }
    y[i] = acc;
  }
  if (sym_lower) {
    for (int64_t i = 0; i < n; ++i) y[i] = y[i] + t[i];
    free(t);
  }
}

/* direct_lu.refactorize (direct_lu.py:297-356) on the factor arrays of LuFactors.
 * avals: general values (to_general order).  Writes Lx, Ux, Udiag in place.
 * diag_out: {max|u|, min|u|, patched, growth}. */
void oracle_refactorize(int64_t n, const int64_t *Ag_rp, const double *avals, int64_t nnz_a,
                        const int64_t *Lp, const int64_t *Li, double *Lx, const int64_t *Up,
                        const int64_t *Ui, double *Ux, double *udiag, const int64_t *so_ptr,
                        const int64_t *so_data, const int64_t *ap_ptr, const int64_t *a_src,
                        const int64_t *a_tgt, double *diag_out) {
  /* eps_patch = 1e-12 * inf_norm(Ag) (:318) */
  double infn = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int64_t p = Ag_rp[i]; p < Ag_rp[i + 1]; ++p) s = s + fabs(avals[p]);
    if (i == 0 || s > infn) infn = s;
  }
  const double eps = 1e-12 * infn;
  double *x = calloc(n ? n : 1, sizeof(double));
  int64_t patched = 0;
  double gmax = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    for (int64_t q = ap_ptr[j]; q < ap_ptr[j + 1]; ++q) x[a_tgt[q]] = avals[a_src[q]];
    for (int64_t t = so_ptr[j]; t < so_ptr[j + 1]; ++t) {
      const int64_t k = so_data[t];
      const double xk = x[k];
      for (int64_t p = Lp[k]; p < Lp[k + 1]; ++p) {
        double prod = Lx[p] * xk;
        x[Li[p]] = x[Li[p]] - prod;
      }
    }
    for (int64_t p = Up[j]; p < Up[j + 1]; ++p) {
      Ux[p] = x[Ui[p]];
      if (fabs(Ux[p]) > gmax) gmax = fabs(Ux[p]);
    }
    double ujj = x[j];
    if (fabs(ujj) > gmax) gmax = fabs(ujj);
    if (fabs(ujj) < eps) {
      ujj = ujj >= 0.0 ? eps : -eps;
      patched++;
    }
    udiag[j] = ujj;
    for (int64_t p = Lp[j]; p < Lp[j + 1]; ++p) {
      if (fabs(x[Li[p]]) > gmax) gmax = fabs(x[Li[p]]);
      Lx[p] = x[Li[p]] / ujj;
    }
    for (int64_t p = Up[j]; p < Up[j + 1]; ++p) x[Ui[p]] = 0.0;
    for (int64_t p = Lp[j]; p < Lp[j + 1]; ++p) x[Li[p]] = 0.0;
    x[j] = 0.0;
  }
  free(x);
  double maxa = 0.0, mx = 0.0, mn = 0.0;
  for (int64_t p = 0; p < nnz_a; ++p)
    if (fabs(avals[p]) > maxa) maxa = fabs(avals[p]);
  for (int64_t j = 0; j < n; ++j) {
    double a = fabs(udiag[j]);
    if (j == 0 || a > mx) mx = a;
    if (j == 0 || a < mn) mn = a;
  }
  diag_out[0] = mx;
  diag_out[1] = mn;
  diag_out[2] = (double)patched;
  diag_out[3] = maxa > 0 ? gmax / maxa : 0.0;
}

/* direct_lu.lu_solve (direct_lu.py:359-379). */
void oracle_lu_solve(int64_t n, const int64_t *row_perm, const int64_t *col_perm, const int64_t *Lp,
                     const int64_t *Li, const double *Lx, const int64_t *Up, const int64_t *Ui,
                     const double *Ux, const double *udiag, const double *b, double *x) {
  double *y = malloc((n ? n : 1) * sizeof(double));
  for (int64_t i = 0; i < n; ++i) y[i] = b[row_perm[i]];
  for (int64_t j = 0; j < n; ++j) {
    const double yj = y[j];
    for (int64_t p = Lp[j]; p < Lp[j + 1]; ++p) {
      double prod = Lx[p] * yj;
      y[Li[p]] = y[Li[p]] - prod;
    }
  }
  for (int64_t j = n - 1; j >= 0; --j) {
    const double wj = y[j] / udiag[j];
    y[j] = wj;
    for (int64_t p = Up[j]; p < Up[j + 1]; ++p) {
      double prod = Ux[p] * wj;
      y[Ui[p]] = y[Ui[p]] - prod;
    }
  }
  for (int64_t i = 0; i < n; ++i) x[col_perm[i]] = y[i];
  free(y);
}

/* ---------------------------------------------------------------------------
 * FGMRES(m) + CGS2 (krylov.py:93-208) with K = spmv(K_lower) and M = lu_solve.
 * Sequential dot products (the reference uses BLAS ddot/dgemv: iteration counts, not
 * bits, are the contract here).
 * ------------------------------------------------------------------------- */
typedef struct {
  int64_t n;
  /* operator */
  const int64_t *k_rp, *k_ci;
  const double *k_v;
  int k_sym;
  /* factors */
  const int64_t *row_perm, *col_perm, *Lp, *Li, *Up, *Ui;
  const double *Lx, *Ux, *udiag;
} oracle_system;

static double dot(int64_t n, const double *a, const double *b) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

static int finite_vec(int64_t n, const double *a) {
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite(a[i])) return 0;
  return 1;
}

/* returns 0 ok, 4 non-finite. out: {iterations, converged, beta0, est_final, true_final} */
int oracle_fgmres(const oracle_system *S, const double *b, const double *x0, int m, int max_outer,
                  double tol, double *x, double *out, double *hist, int hist_cap) {
  const int64_t n = S->n;
  double *V = malloc(sizeof(double) * (size_t)(m + 1) * (n ? n : 1));
  double *Z = malloc(sizeof(double) * (size_t)m * (n ? n : 1));
  double *w = malloc(sizeof(double) * (n ? n : 1)), *r = malloc(sizeof(double) * (n ? n : 1));
  double *H = calloc((size_t)(m + 1) * m, sizeof(double));
  double *cs = calloc(m + 1, sizeof(double)), *sn = calloc(m + 1, sizeof(double));
  double *g = calloc(m + 1, sizeof(double)), *yv = calloc(m + 1, sizeof(double));
  double *h = calloc(m + 1, sizeof(double)), *h2 = calloc(m + 1, sizeof(double));
  int rc = 0, hn = 0;
  memcpy(x, x0, sizeof(double) * n);
  oracle_spmv(n, S->k_rp, S->k_ci, S->k_v, S->k_sym, x, r);
  if (!finite_vec(n, r)) { rc = 4; goto done; }
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
  double beta0 = sqrt(dot(n, r, r));
  if (hist && hn < hist_cap) hist[hn] = beta0;
  hn++;
  out[2] = beta0;
  int iters = 0, converged = 0;
  double beta = beta0, est = beta0;
  if (beta0 == 0.0) {
    converged = 1;
    beta = 0.0;
    goto fin;
  }
  const double target = tol * beta0, floor_ = 1e-14 * beta0;
  for (int outer = 0; outer < max_outer; ++outer) {
    if (beta <= target) { converged = 1; break; }
    for (int64_t i = 0; i < n; ++i) V[i] = r[i] / beta;
    memset(H, 0, sizeof(double) * (size_t)(m + 1) * m);
    memset(g, 0, sizeof(double) * (m + 1));
    g[0] = beta;
    int j_used = 0, stop = 0;
    for (int j = 0; j < m; ++j) {
      double *Vj = V + (size_t)j * n, *Zj = Z + (size_t)j * n;
      oracle_lu_solve(n, S->row_perm, S->col_perm, S->Lp, S->Li, S->Lx, S->Up, S->Ui, S->Ux,
                      S->udiag, Vj, Zj);
      if (!finite_vec(n, Zj)) { rc = 4; goto done; }
      oracle_spmv(n, S->k_rp, S->k_ci, S->k_v, S->k_sym, Zj, w);
      if (!finite_vec(n, w)) { rc = 4; goto done; }
      for (int pass = 0; pass < 2; ++pass) { /* cgs2_step (krylov.py:93-105) */
        double *hh = pass ? h2 : h;
        for (int q = 0; q <= j; ++q) hh[q] = dot(n, V + (size_t)q * n, w);
        for (int64_t i = 0; i < n; ++i) {
          double t = 0.0;
          for (int q = 0; q <= j; ++q) t += V[(size_t)q * n + i] * hh[q];
          w[i] = w[i] - t;
        }
      }
      for (int q = 0; q <= j; ++q) H[q * m + j] = h[q] + h2[q];
      const double hj1 = sqrt(dot(n, w, w));
      H[(j + 1) * m + j] = hj1;
      for (int i = 0; i < j; ++i) {
        double a = H[i * m + j], bb = H[(i + 1) * m + j];
        double t = cs[i] * a + sn[i] * bb;
        H[(i + 1) * m + j] = -sn[i] * a + cs[i] * bb;
        H[i * m + j] = t;
      }
      double denom = hypot(H[j * m + j], H[(j + 1) * m + j]);
      cs[j] = H[j * m + j] / denom;
      sn[j] = H[(j + 1) * m + j] / denom;
      H[j * m + j] = denom;
      H[(j + 1) * m + j] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      est = fabs(g[j + 1]);
      if (hist && hn < hist_cap) hist[hn] = est;
      hn++;
      iters++;
      j_used = j + 1;
      if (est <= target || hj1 <= floor_) { stop = 1; break; }
      for (int64_t i = 0; i < n; ++i) V[(size_t)(j + 1) * n + i] = w[i] / hj1;
    }
    for (int i = j_used - 1; i >= 0; --i) { /* _solve_upper (krylov.py:211-216) */
      double d = 0.0;
      for (int q = i + 1; q < j_used; ++q) d += H[i * m + q] * yv[q];
      yv[i] = (g[i] - d) / H[i * m + i];
    }
    for (int64_t i = 0; i < n; ++i) {
      double t = 0.0;
      for (int q = 0; q < j_used; ++q) t += Z[(size_t)q * n + i] * yv[q];
      x[i] = x[i] + t;
    }
    oracle_spmv(n, S->k_rp, S->k_ci, S->k_v, S->k_sym, x, r);
    if (!finite_vec(n, r)) { rc = 4; goto done; }
    for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
    beta = sqrt(dot(n, r, r));
    if (stop) { converged = 1; break; }
    if (beta <= target) { converged = 1; break; }
  }
fin:
  out[0] = iters;
  out[1] = converged;
  out[3] = est;
  out[4] = beta;
done:
  free(V); free(Z); free(w); free(r); free(H); free(cs); free(sn); free(g); free(yv); free(h);
  free(h2);
  return rc;
}

/* refine.refine_fgmres (refine.py:103-132).  out: {triggered, iterations, converged,
 * nsr_before, nsr_after, rr_est} */
int oracle_refine_fgmres(const oracle_system *S, const double *r, const double *x0, int m,
                         int max_outer, double delta, double *x, double *out) {
  const int64_t n = S->n;
  double *t = malloc(sizeof(double) * (n ? n : 1));
  oracle_spmv(n, S->k_rp, S->k_ci, S->k_v, S->k_sym, x0, t);
  double e2 = 0.0, r2 = 0.0, emax = 0.0, xmax = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double e = r[i] - t[i];
    e2 += e * e;
    r2 += r[i] * r[i];
    if (fabs(e) > emax) emax = fabs(e);
    if (fabs(x0[i]) > xmax) xmax = fabs(x0[i]);
  }
  const double kinf = oracle_inf_norm(n, S->k_rp, S->k_ci, S->k_v, S->k_sym);
  const double nsr0 = (kinf * xmax) == 0.0 ? INFINITY : emax / (kinf * xmax);
  memset(out, 0, 6 * sizeof(double));
  out[3] = nsr0;
  int rc = 0;
  if (!(sqrt(e2) > delta * sqrt(r2))) {
    memcpy(x, x0, sizeof(double) * n);
    out[2] = 1;
    out[4] = nsr0;
    out[5] = 1.0;
  } else {
    double fo[5] = {0, 0, 0, 0, 0};
    rc = oracle_fgmres(S, r, x0, m, max_outer, delta, x, fo, NULL, 0);
    out[0] = 1;
    out[1] = fo[0];
    out[2] = fo[1];
    out[5] = fo[2] > 0 ? fo[3] / fo[2] : 0.0;
    oracle_spmv(n, S->k_rp, S->k_ci, S->k_v, S->k_sym, x, t);
    emax = 0.0;
    xmax = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      double e = fabs(r[i] - t[i]);
      if (e > emax) emax = e;
      if (fabs(x[i]) > xmax) xmax = fabs(x[i]);
    }
    out[4] = (kinf * xmax) == 0.0 ? INFINITY : emax / (kinf * xmax);
  }
  free(t);
  return rc;
}
