"""Reference goldens at the BASELINE configuration sizes (run in the build container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_large.py CASE [CASE ...]

CASE is one of ``activsg200`` (N = 9,030, configs[0]), ``activsg200p`` (the same family with
imbalance slacks on half the buses: the reference's threshold pivoting then picks ~1,400
off-diagonal pivots), ``activsg2000`` (N = 90,320, configs[1]) and ``activsg2000p``
(imbalance slacks on 75 % of the buses: ~7,600 off-diagonal pivots, fill ~10x, 1.9 G update
pairs per refactorization) and ``activsg2000q`` (90 %: ~3,200 off-diagonal pivots, fill ~2.6x).

For each case the REFERENCE package (``kktsolve`` imported from /root/reference, never needed
at test time) runs exactly the hot path of ``harness._run_direct_family`` (harness.py:217-269):
``factorize`` of system 0 (direct_lu.py:116-294), then per system k = 0..19
``refactorize`` (:297-356) -> ``lu_solve`` (:359-379) -> ``refine_fgmres`` (refine.py:103-132)
at the fixed delta = 1e-10 and at the barrier-tied delta(mu_k) of ``refine.BarrierTiedTolerance``.

What is stored (``<case>.npz``): the analysis arrays in full for the 9k cases and as SHA-256
digests for the 90k cases (``sha_<array>``, over the little-endian int64 / float64 bytes); per
system the LuDiagnostics, SHA-256 of the refactorized ``_Lx/_Ux/_Udiag`` and of ``x0``; the full
x0 / refined x of a few systems; and the refine reports.  The fixture generator is
``acopf.make_sequence`` (pure numpy, deterministic from the seed), so the tests rebuild the
inputs and only the reference's outputs need to be stored.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

from kktsolve import direct_lu as R_lu  # noqa: E402
from kktsolve import sparsecore as R_sc  # noqa: E402
from kktsolve.krylov import KrylovConfig  # noqa: E402
from kktsolve.refine import RefinementConfig, refine_fgmres  # noqa: E402

import paper_2401_13926_b200.acopf as acopf  # noqa: E402  (pure numpy generator)
from paper_2401_13926_b200.refine import BarrierTiedTolerance  # noqa: E402  (pure policy)

# case -> (acopf config, imbalance_frac, store full arrays, systems whose full x0 / x are kept)
CASES = {
    "activsg200": ("activsg200", 1.0, True, (1, 10, 19)),
    "activsg200p": ("activsg200", 0.5, True, (1, 10, 19)),
    "activsg2000": ("activsg2000", 1.0, False, (19,)),
    "activsg2000p": ("activsg2000", 0.75, False, (19,)),
    "activsg2000q": ("activsg2000", 0.9, False, (19,)),
}
M = 20
FACTOR_KEYS = ["row_perm", "col_perm", "Lp", "Li", "Lx", "Up", "Ui", "Ux", "Udiag", "so_ptr",
               "so_data", "ap_ptr", "a_src", "a_tgt"]
REPORT_KEYS = ["triggered", "ir_iterations", "triangular_solves_used", "nsr_before", "nsr_after",
               "rr_final", "nrbe_final", "converged"]


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    a = a.astype(np.float64 if a.dtype.kind == "f" else np.int64, copy=False)
    return hashlib.sha256(a.tobytes()).hexdigest()


def factor_arrays(f) -> dict:
    return dict(row_perm=f.row_perm.perm, col_perm=f.col_perm.perm, Lp=f._Lp, Li=f._Li,
                Lx=f._Lx, Up=f._Up, Ui=f._Ui, Ux=f._Ux, Udiag=f._Udiag, so_ptr=f._so_ptr,
                so_data=f._so_data, ap_ptr=f._ap_ptr, a_src=f._a_src, a_tgt=f._a_tgt)


def run(case: str) -> None:
    cfg, frac, full, keep = CASES[case]
    seq = acopf.make_sequence(cfg, seed=0, length=M, imbalance_frac=frac)
    P = seq.pattern.K
    Ks = [R_sc.CsMatrix(P.n_rows, P.n_cols, P.row_ptr, P.col_idx, seq.values(k),
                        R_sc.SYMMETRIC_LOWER) for k in range(M)]
    out: dict = {"n": np.array([P.n_rows]), "nnz_lower": np.array([P.nnz]),
                 "imbalance_frac": np.array([frac])}
    t0 = time.time()
    f, d0 = R_lu.factorize(R_sc.to_general(Ks[0]))
    t_fact = time.time() - t0
    for k, v in factor_arrays(f).items():
        if full:
            out[f"f0_{k}"] = np.array(v, copy=True)
        out[f"sha_{k}"] = np.array(sha(v))
    out["f0_diag"] = np.array([d0.max_abs_pivot, d0.min_abs_pivot, d0.zero_pivots_patched,
                               d0.growth_estimate])
    out["offdiag_pivots"] = np.array([int(np.sum(f.row_perm.perm != f.col_perm.perm))])
    policy = BarrierTiedTolerance()
    diags, sh_fact, sh_x0 = [], [], []
    reps = {"1e-10": [], "barrier": []}
    deltas_barrier = []
    t_ref = t_solve = t_refine = 0.0
    for k in range(M):
        K = Ks[k]
        r = seq.rhs(k)
        t = time.time()
        d = R_lu.refactorize(f, R_sc.to_general(K))
        t_ref += time.time() - t
        diags.append([d.max_abs_pivot, d.min_abs_pivot, d.zero_pivots_patched, d.growth_estimate])
        sh_fact.append([sha(f._Lx), sha(f._Ux), sha(f._Udiag)])
        t = time.time()
        x0 = R_lu.lu_solve(f, r)
        t_solve += time.time() - t
        sh_x0.append(sha(x0))
        if k in keep:
            out[f"s{k}_x0"] = x0
        db = policy(seq.mu(k))
        deltas_barrier.append(db)
        for tag, delta in (("1e-10", 1e-10), ("barrier", db)):
            t = time.time()
            x, rep = refine_fgmres(K, f, x0, r, RefinementConfig(delta_tol=delta,
                                                                 krylov=KrylovConfig(m=10)))
            t_refine += time.time() - t
            rr = float(np.linalg.norm(r - R_sc.spmv(K, x)) / np.linalg.norm(r))
            reps[tag].append([float(getattr(rep, key)) for key in REPORT_KEYS] + [rr])
            if k in keep:
                out[f"s{k}_x_{tag}"] = x
        print(case, "k", k, "iters", reps["1e-10"][-1][1], reps["barrier"][-1][1], flush=True)
    out["refactor_diag"] = np.array(diags)
    out["sha_factors"] = np.array(sh_fact)
    out["sha_x0"] = np.array(sh_x0)
    out["delta_barrier"] = np.array(deltas_barrier)
    for tag, rows in reps.items():
        out[f"refine_{tag}"] = np.array(rows)
    out["report_keys"] = np.array(REPORT_KEYS + ["rr_true"])
    out["seconds"] = np.array([t_fact, t_ref, t_solve, t_refine])
    np.savez_compressed(os.path.join(HERE, f"large_{case}.npz"), **out)
    meta = dict(reference="/root/reference/pkg (kktsolve 0.1.0)", numpy=np.__version__,
                      n=int(P.n_rows), nnz_L=int(f._Li.size), nnz_U=int(f._Ui.size),
                      offdiag_pivots=int(out["offdiag_pivots"][0]),
                      seconds=dict(factorize=t_fact, refactorize=t_ref, lu_solve=t_solve,
                                   refine=t_refine))
    with open(os.path.join(HERE, f"large_{case}.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print(case, "done", meta, flush=True)


if __name__ == "__main__":
    for c in sys.argv[1:] or list(CASES):
        run(c)
