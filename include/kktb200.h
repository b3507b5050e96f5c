/*
 * kktb200.h — C ABI of the B200-native KKT refactor / solve / FGMRES-IR hot path.
 *
 * One shared library, libkktb200.so, built from
 *   paper_2401_13926_b200/csrc/analyze.cpp   (host: ordering + first pivoted LU, bit-exact)
 *   paper_2401_13926_b200/csrc/device.cu     (sm_100a kernels + device handle)
 *
 * Plain C types only (no torch, no STL) so any FFI (ctypes, cffi, cgo, JNI) can bind it.
 * Every entry point returns an int status (KKT_OK == 0); kkt_last_error() gives the
 * thread-local message of the last failure.  The Python facade maps the codes 1:1 to the
 * reference's exception classes.
 *
 * Reference interfaces replaced (paths relative to the reference package
 * pkg/src/kktsolve/):
 *   kkt_analyze            <- direct_lu.factorize(A, pivot_tol)          direct_lu.py:116
 *                             (+ ordering.min_degree_order               ordering.py:19)
 *   kkt_symbolic_export    <- the LuFactors hand-off object               direct_lu.py:51-81
 *   kkt_dev_refactor       <- direct_lu.refactorize(factors, A_new)      direct_lu.py:297
 *   kkt_dev_solve          <- direct_lu.lu_solve(factors, b)             direct_lu.py:359
 *   kkt_dev_spmv           <- sparsecore.spmv(K, x)                      sparsecore.py:284
 *   kkt_dev_residual_norms <- refine.nsr / nrbe / needs_refinement       refine.py:62-92
 *   kkt_dev_fgmres         <- krylov.fgmres(K, M=lu_solve, b, x0, cfg)   krylov.py:117
 *   kkt_dev_fgmres_ops     <- krylov.fgmres(K, M, b, x0, cfg) for any LinearOperator pair
 *                             (matrix / identity / LU / host callback)   krylov.py:36-54,117
 *   kkt_dev_refine_fgmres  <- refine.refine_fgmres(K, f, x0, r, cfg)     refine.py:103
 *   kkt_dev_residual       <- rho = r - spmv(K, x); ||rho||_2            refine.py:158,167-168
 *   kkt_dev_axpy           <- x += d  (Richardson update)                refine.py:166
 *   kkt_assemble_values    <- kkt.assemble_kkt values (frozen pattern)   kkt.py:88-124
 *   kkt_assemble_rhs       <- kkt.assemble_rhs                           kkt.py:127-137
 *   kkt_recover_dz         <- kkt.recover_dz                             kkt.py:140-144
 *   kkt_mm_info / kkt_mm_read_coo / kkt_mm_read_array
 *                          <- mmio.load_matrix_market / load_vector      mmio.py:36-130
 */
#ifndef KKTB200_H
#define KKTB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mirrored by the facade's exception mapping) ---- */
enum {
  KKT_OK = 0,
  KKT_ERR_SINGULAR = 1,         /* SingularMatrixError        direct_lu.py:35  */
  KKT_ERR_PATTERN_MISMATCH = 2, /* PatternMismatchError       direct_lu.py:39  */
  KKT_ERR_BAD_SHAPE = 3,        /* ValueError (shape / argument)               */
  KKT_ERR_NONFINITE = 4,        /* OperatorOutputError        krylov.py:28     */
  KKT_ERR_CUDA = 5,             /* CUDA runtime failure                        */
  KKT_ERR_OOM = 6,              /* allocation failure                          */
  KKT_ERR_BAD_ARG = 7,          /* ValueError (config validation)              */
  KKT_ERR_CALLBACK = 8          /* a host operator callback reported failure   */
};

const char *kkt_last_error(void);
int kkt_abi_version(void);

/* ======================================================================
 * Host analysis (stays on the CPU, bit-exact with the reference).
 * ====================================================================== */
typedef struct kkt_symbolic kkt_symbolic;

/* Sizes reported by kkt_symbolic_sizes(), in this order. */
enum {
  KKT_SZ_N = 0,   /* n                                   */
  KKT_SZ_NNZ_A,   /* nnz of the general input pattern    */
  KKT_SZ_NNZ_L,   /* strict L entries  (_Li/_Lx)         */
  KKT_SZ_NNZ_U,   /* strict U entries  (_Ui/_Ux)         */
  KKT_SZ_NSO,     /* replay schedule   (_so_data)        */
  KKT_SZ_NAP,     /* A-scatter map     (_a_src/_a_tgt)   */
  KKT_SZ_COUNT
};

/* factorize(): A is GENERAL CSR (row_ptr[n+1], col_idx[nnz] sorted+unique per row,
 * values[nnz]).  Runs min_degree_order + left-looking Gilbert-Peierls LU with threshold
 * partial pivoting (pivot_tol in (0,1]) exactly as direct_lu.py:116-294.
 * On KKT_ERR_SINGULAR, *out is NULL and kkt_last_error() names the column. */
int kkt_analyze(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                const double *values, double pivot_tol, kkt_symbolic **out);

/* Ordering only: min_degree_order(A) (ordering.py:19-59) -> perm[n]. */
int kkt_min_degree_order(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                         int64_t *perm_out);

void kkt_symbolic_free(kkt_symbolic *s);
int kkt_symbolic_sizes(const kkt_symbolic *s, int64_t sizes[KKT_SZ_COUNT]);

/* Copy the LuFactors arrays out (caller allocates with the reported sizes).
 * Any pointer may be NULL to skip that array. */
int kkt_symbolic_export(const kkt_symbolic *s, int64_t *row_perm, int64_t *col_perm,
                        int64_t *Lp, int64_t *Li, double *Lx,
                        int64_t *Up, int64_t *Ui, double *Ux, double *Udiag,
                        int64_t *so_ptr, int64_t *so_data,
                        int64_t *ap_ptr, int64_t *a_src, int64_t *a_tgt);

/* LuDiagnostics of the first factorization: {max|u_jj|, min|u_jj|, patched, growth}. */
int kkt_symbolic_diag(const kkt_symbolic *s, double diag[4]);

/* Schedule statistics: {refactor levels, L-solve levels, U-solve levels,
 * refactor update pairs (F/2), max |so(j)|, max L col, max U col, max L row, max U row}. */
int kkt_symbolic_stats(const kkt_symbolic *s, int64_t stats[9]);

/* ======================================================================
 * Device handle: one GPU, one stream, all buffers allocated once.
 * Calls on one handle must be serialised by the caller.  Handles on different GPUs may run
 * concurrently; handles on the SAME GPU must not: the refactorization and grid-solve
 * kernels are persistent, sync-free grids sized to the GPU's resident-CTA capacity, so two
 * of them running side by side are not guaranteed co-resident.
 * ====================================================================== */
typedef struct kkt_device kkt_device;

/* Input value layout for kkt_dev_refactor / operator values. */
enum { KKT_LAYOUT_GENERAL = 0, KKT_LAYOUT_SYMMETRIC_LOWER = 1 };

typedef struct {
  int device;             /* CUDA ordinal                                  */
  int batch;              /* number of same-pattern systems held (>=1)     */
  int restart_m;          /* FGMRES restart length the workspace is sized for */
  int reserved;           /* 0 (the solves are always bitwise with lu_solve) */
  int flags;              /* reserved, 0                                   */
} kkt_device_opts;

/* Create the device handle from the host analysis.  A_row_ptr/A_col_idx repeat the
 * general pattern that was analysed (checked).  lower_nnz / gen_src (optional, may be
 * 0 / NULL) describe the symmetric-lower storage of the same matrix: general entry e holds
 * lower value gen_src[e] (the to_general map, sparsecore.py:263-273).  With it, values may
 * be passed in KKT_LAYOUT_SYMMETRIC_LOWER (half the upload) and the operator is applied in
 * the reference's symmetric-lower spmv order (sparsecore.py:296-302). */
int kkt_dev_create(const kkt_symbolic *s, const int64_t *A_row_ptr, const int64_t *A_col_idx,
                   int64_t lower_nnz, const int64_t *gen_src, const kkt_device_opts *opts,
                   kkt_device **out);
void kkt_dev_destroy(kkt_device *d);

/* Host-only check of the execution plan kkt_dev_create would build (no GPU needed): the
 * single-system grid phases' chain task lists.  out = {tasks L, tasks U, chains, chain rows,
 * longest chain, order violations, coverage violations, 0}.  Zero order violations means
 * every task reads only values published by tasks earlier in its list, which is what makes
 * the persistent, sync-free grid deadlock-free.  Test/diagnostic entry, no reference
 * counterpart. */
int kkt_plan_check(const kkt_symbolic *s, const int64_t *A_row_ptr, const int64_t *A_col_idx,
                   int64_t lower_nnz, const int64_t *gen_src, int64_t out[8]);

/* Raw CUDA stream (cudaStream_t) the handle launches on. */
void *kkt_dev_stream(kkt_device *d);

/* Upload new values (host or device pointer; nnz doubles of the given layout) and
 * refactorize on the frozen schedule (direct_lu.py:297-356).  The same values become the
 * operator of kkt_dev_spmv / fgmres (general layout => general spmv order).
 * diag_out (host, may be NULL) receives {max|u|, min|u|, patched, growth}. */
int kkt_dev_refactor(kkt_device *d, const double *values_in, int layout, int values_on_device,
                     double *diag_out);

/* Operator-only value update (SpMV / FGMRES operator) without refactorizing. */
int kkt_dev_set_operator_values(kkt_device *d, const double *values_in, int layout,
                                int values_on_device);

/* x = lu_solve(b) (direct_lu.py:359-379).  b, x: n*batch doubles, device pointers. */
int kkt_dev_solve(kkt_device *d, const double *b_dev, double *x_dev);

/* y = K x on the operator values (sparsecore.py:284-305).  Device pointers. */
int kkt_dev_spmv(kkt_device *d, const double *x_dev, double *y_dev);

/* Residual statistics for r - K x (device pointers, batch systems):
 * out[batch][6] = {||r-Kx||_2, ||r-Kx||_inf, ||x||_2, ||x||_inf, ||r||_2, ||K||_inf}. */
int kkt_dev_residual_norms(kkt_device *d, const double *r_dev, const double *x_dev,
                           double *out_host);

/* rho = r - K x (the reference's spmv order, then the subtraction) and norms_host[batch] =
 * ||rho||_2 per system: the Richardson residual (refine.py:158,167-168).  Device vectors. */
int kkt_dev_residual(kkt_device *d, const double *r_dev, const double *x_dev, double *rho_dev,
                     double *norms_host);

/* Matrix Market ingestion (host, C++; mmio.py:36-130).  kkt_mm_info: info[5] = {format
 * (0 coordinate, 1 array), symmetric, rows, cols, nnz (array: rows)}.  kkt_mm_read_coo: the
 * coordinate entries, 0-based, in file order (triplets; symmetric files: lower triangle).
 * kkt_mm_read_array: an n x 1 array file.  Errors carry "path:line: message". */
int kkt_mm_info(const char *path, int64_t *info);
int kkt_mm_read_coo(const char *path, int64_t nnz, int64_t *rows, int64_t *cols, double *vals);
int kkt_mm_read_array(const char *path, int64_t n, double *out);

/* Interior-point bookkeeping on the device (kkt.py:88-144), nb systems, system-major
 * device arrays, run on `stream` (a cudaStream_t, may be NULL).
 * kkt_assemble_values: K[nb][nnz_K] of the frozen symmetric-lower pattern; position p sums
 *   its sources src[p][0..1] (int32 pairs, -1 = none) in order: ids 0..nH-1 = H values,
 *   nH..nH+n-1 = D_x = z/x diagonal, nH+n.. = J values (np.add.at order, kkt.py:104-107).
 * kkt_assemble_rhs: rhs[nb][n+m] = [r~_x + (z - mu/x); r_lambda], mu[nb] on the device.
 * kkt_recover_dz: dz[nb][n] = (r_z - z*dx)/x, dx of system s at dx + s*dx_stride. */
int kkt_assemble_values(int64_t nnz_K, int64_t n, int64_t nH, int64_t nJ, int nb,
                        const int32_t *src_dev, const double *H_dev, const double *J_dev,
                        const double *x_dev, const double *z_dev, double *K_dev, void *stream);
int kkt_assemble_rhs(int64_t n, int64_t m, int nb, const double *r_tilde_x, const double *r_lambda,
                     const double *x, const double *z, const double *mu_dev, double *rhs, void *stream);
int kkt_recover_dz(int64_t n, int nb, int64_t dx_stride, const double *r_z, const double *z,
                   const double *dx, const double *x, double *dz, void *stream);

/* x += y elementwise over the handle's n * batch entries (refine.py:166).  Device vectors. */
int kkt_dev_axpy(kkt_device *d, double *x_dev, const double *y_dev);

typedef struct {
  int m;                  /* restart length                  (krylov.py:61) */
  int max_outer;          /* restart cycles                  (krylov.py:62) */
  double tol;             /* relative tolerance              (krylov.py:63) */
  double delta_tol;       /* refinement trigger (refine only; refine.py:35) */
  const double *delta_sys; /* optional per-system delta_tol (and tol) [batch], or NULL:
                              each system of a batch may carry its own barrier parameter */
  int flags;              /* KKT_FG_* below                                  */
} kkt_krylov_cfg;

enum {
  KKT_FG_STATS_AFTER = 1, /* refine: also compute the residual statistics of the result   */
  KKT_FG_HOST_LOOP = 2,   /* drive the restart/iteration control from the host (reads the
                             device control words per iteration) instead of one CUDA graph
                             with conditional nodes; same kernels, same results          */
  KKT_FG_MGS = 4,         /* modified Gram-Schmidt (KrylovConfig.ortho = "mgs") instead of
                             CGS2                                                        */
  KKT_FG_NO_HANDOFF = 8   /* batched handles: keep every system in the lockstep batch to
                             the end (default: once at most min(4, batch/16) systems still
                             run, they finish on single-system helper handles)            */
};

typedef struct {
  int iterations;         /* KrylovResult.iterations          */
  int converged;          /* KrylovResult.converged           */
  int precond_applications;
  int restarts;           /* number of restart cycles run      */
  double beta0;           /* est_residual_history[0]           */
  double est_final;       /* est_residual_history[-1]          */
  double true_final;      /* KrylovResult.true_final_residual  */
  int triggered;          /* refine only                       */
  int nonfinite;          /* a NaN/Inf was produced: this system failed (OperatorOutputError) */
  double stats_before[6]; /* refine: {||r-Kx0||_2, ||r-Kx0||_inf, ||x0||_2, ||x0||_inf,
                             ||r||_2, ||K||_inf}  (nsr_before, refine.py:117)         */
  double stats_after[6];  /* refine + KKT_FG_STATS_AFTER: the same for the returned x
                             (nsr_after / nrbe_final, refine.py:129-131)             */
  int handed_off;         /* batched handles: this straggler's last iterations ran on a
                             single-system helper (same arithmetic; KKT_HANDOFF)       */
  int reserved_;
} kkt_krylov_report;

/* FGMRES(m) with CGS2, K = operator values, M = lu_solve with the current factors
 * (krylov.py:117-208).  Device pointers; batch==1.  history_host (may be NULL) gets
 * up to hist_cap estimated residuals (est_residual_history). */
int kkt_dev_fgmres(kkt_device *d, const double *b_dev, const double *x0_dev, double *x_dev,
                   const kkt_krylov_cfg *cfg, kkt_krylov_report *rep,
                   double *history_host, int hist_cap);

/* Operators of the generic FGMRES (krylov.LinearOperator, krylov.py:36-54).
 * KKT_OP_HANDLE: K = the handle's operator values (spmv), M = its LU factors (lu_solve);
 * KKT_OP_IDENTITY: v -> v (LinearOperator.identity); KKT_OP_MATRIX: a kkt_operator's spmv;
 * KKT_OP_CALLBACK: apply(user, in_host, out_host) — host code (the reference's numpy
 * callback) that reads n doubles from in_host and writes n doubles to out_host (library-owned
 * pinned buffers) and returns 0.  Non-HANDLE kinds need batch == 1. */
typedef int (*kkt_apply_fn)(void *user, const double *in_host, double *out_host);
enum { KKT_OP_HANDLE = 0, KKT_OP_IDENTITY = 1, KKT_OP_MATRIX = 2, KKT_OP_CALLBACK = 3 };
typedef struct kkt_operator kkt_operator;
typedef struct {
  int kind;
  kkt_operator *matrix;   /* KKT_OP_MATRIX */
  kkt_apply_fn apply;     /* KKT_OP_CALLBACK */
  void *user;
} kkt_linop;

/* fgmres(K, M, b, x0, cfg) (krylov.py:117-208) with any operator pair.  Device vectors.
 * history_host[hist_cap] (may be NULL): est_residual_history; restart_pairs_host
 * [pairs_cap][2] (may be NULL): KrylovResult.restart_residuals (krylov.py:193). */
int kkt_dev_fgmres_ops(kkt_device *d, const kkt_linop *K, const kkt_linop *M, const double *b_dev,
                       const double *x0_dev, double *x_dev, const kkt_krylov_cfg *cfg,
                       kkt_krylov_report *rep, double *history_host, int hist_cap,
                       double *restart_pairs_host, int pairs_cap);

/* refine_fgmres (refine.py:103-132): trigger on ||r-Kx0||_2 > delta*||r||_2, then
 * FGMRES with tol = delta_tol.  Device pointers. */
int kkt_dev_refine_fgmres(kkt_device *d, const double *r_dev, const double *x0_dev,
                          double *x_dev, const kkt_krylov_cfg *cfg, kkt_krylov_report *rep);

/* The whole per-system hot path of harness._run_direct_family (harness.py:223-245):
 * refactor(values) -> x0 = solve(r) -> refine_fgmres.  values/r on host or device. */
int kkt_dev_step(kkt_device *d, const double *values_in, int layout, const double *r_in,
                 double *x_out, int io_on_device, const kkt_krylov_cfg *cfg,
                 kkt_krylov_report *rep, double *diag_out);

/* The second half of kkt_dev_step for factors already refactorized (kkt_dev_refactor):
 * x0 = solve(r) -> refine_fgmres -> x.  Lets a caller overlap the rhs upload with the
 * refactorization (pipeline.BatchPipeline).  r/x on host or device. */
int kkt_dev_step_solve(kkt_device *d, const double *r_in, double *x_out, int io_on_device,
                       const kkt_krylov_cfg *cfg, kkt_krylov_report *rep);

/* Download the current factor values in the LuFactors layout (_Lx, _Ux, _Udiag). */
int kkt_dev_download_factors(kkt_device *d, double *Lx, double *Ux, double *Udiag);

/* The inverse (batch == 1): make (_Lx, _Ux, _Udiag) the handle's current factors, e.g. to
 * re-create a device handle for LuFactors whose values came from an earlier refactorize. */
int kkt_dev_upload_factors(kkt_device *d, const double *Lx, const double *Ux, const double *Udiag);

/* ======================================================================
 * Standalone operator (sparsecore.spmv / refine.nsr / refine.nrbe on a bare matrix).
 * row_ptr/col_idx: CSR as stored (symmetric_lower != 0 => lower triangle incl. diagonal,
 * applied with both halves exactly like sparsecore.py:296-302).
 * ====================================================================== */
int kkt_op_create(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                  int symmetric_lower, int device, kkt_operator **out);
void kkt_op_destroy(kkt_operator *op);
void *kkt_op_stream(kkt_operator *op);
int kkt_op_set_values(kkt_operator *op, const double *values, int values_on_device);
int kkt_op_spmv(kkt_operator *op, const double *x_dev, double *y_dev);
/* out6 as kkt_dev_residual_norms */
int kkt_op_residual_norms(kkt_operator *op, const double *r_dev, const double *x_dev,
                          double *out_host);

/* Schedule of the handle: {n, pL, pU, L grid levels, U grid levels, L tail rows, U head rows,
 * refactor blocks, refactor warps/block, refactor smem bytes, trisolve grid blocks,
 * refactor levels, arena bytes, update pairs, 0, 0}. */
int kkt_dev_info(kkt_device *d, int64_t info[16]);

/* Timeline of the last refactor / solve when the handle was created with KKT_TRACE=1:
 * refactor_out[2n] = {dispatch ns, done ns} per column, trisolve_out[2n] = publish ns per
 * row of the L then the U sweep (grid phase rows).  Profiling aid. */
int kkt_dev_trace(kkt_device *d, uint64_t *refactor_out, uint64_t *trisolve_out);
/* Secondary trace buffer, max(n_so, 4n) entries: single system — ns when each replay step
 * (so entry) of the last refactor was applied (bit 0: it was late); batch — per-warp cycle
 * counters of k_b_refactor and {start, critical-dependency ready} ns per grid-phase row of
 * the last solve (system 0; L rows at 2r, U rows at 2(n+r)).  Profiling aid. */
int kkt_dev_trace_steps(kkt_device *d, uint64_t *steps_out);

/* Kernel launches issued by this handle since creation (evidence counter). */
int64_t kkt_dev_launch_count(kkt_device *d);

/* kkt_dev_solve / kkt_dev_spmv on vectors in the handle's INTERNAL layout (batched handles:
 * [n][nbp] interleaved, nbp = batch rounded up to 32; single: [n]) — the kernels without the
 * boundary transposes, for per-kernel timing (bench.py roofline). */
int kkt_dev_solve_native(kkt_device *d, const double *b_dev, double *x_dev);
int kkt_dev_spmv_native(kkt_device *d, const double *x_dev, double *y_dev);

/* Measurement probe (bench.py's critical-path bound; no reference counterpart): the latency of
 * one dependency hop between SMs — a value published with a relaxed 64-bit store and observed
 * by a relaxed poll on another SM — averaged over `rounds` ping-pong round trips. */
int kkt_probe_hop_ns(int device, int rounds, double *ns_per_hop);

#ifdef __cplusplus
}
#endif
#endif /* KKTB200_H */
