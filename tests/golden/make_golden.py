"""Generate the golden fixtures from the REFERENCE implementation (run in the build container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports the reference package ``kktsolve`` from /root/reference (read-only; never needed at
test time) and records, for small inputs, exactly what its hot path produces:
factorize arrays, refactorize values (bitwise), lu_solve / spmv outputs (bitwise),
refine_fgmres reports and harness rows.  The GPU parity tests and the oracle self-tests
compare against these files; /root/reference does not exist on the GPU box.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, ROOT)

from kktsolve import direct_lu as R_lu  # noqa: E402
from kktsolve import sparsecore as R_sc  # noqa: E402
from kktsolve.harness import (MatrixSequence, SequenceItem, StrategySpec,  # noqa: E402
                              run_strategy, sequence_from_trace)
from kktsolve.krylov import KrylovConfig  # noqa: E402
from kktsolve.refine import RefinementConfig, refine_fgmres, refine_richardson  # noqa: E402
from kktsolve.seqgen import standard_trace  # noqa: E402
from conftest import random_sparse  # noqa: E402  (reference test generator)

import paper_2401_13926_b200.acopf as acopf  # noqa: E402  (pure numpy generator)

FACTOR_KEYS = ["row_perm", "col_perm", "Lp", "Li", "Lx", "Up", "Ui", "Ux", "Udiag", "so_ptr",
               "so_data", "ap_ptr", "a_src", "a_tgt"]


def factor_arrays(f) -> dict:
    return dict(row_perm=f.row_perm.perm, col_perm=f.col_perm.perm, Lp=f._Lp, Li=f._Li,
                Lx=f._Lx.copy(), Up=f._Up, Ui=f._Ui, Ux=f._Ux.copy(), Udiag=f._Udiag.copy(),
                so_ptr=f._so_ptr, so_data=f._so_data, ap_ptr=f._ap_ptr, a_src=f._a_src,
                a_tgt=f._a_tgt)


def diag_vec(d) -> np.ndarray:
    return np.array([d.max_abs_pivot, d.min_abs_pivot, d.zero_pivots_patched, d.growth_estimate])


def sequence_case(name, Ks, rhss, deltas=(1e-10, 1e-14), keep_factor_vals=None):
    """Ks: list of reference CsMatrix (symmetric-lower, shared pattern)."""
    out = {}
    K0 = Ks[0]
    out["n"] = np.array([K0.n_rows])
    out["K_row_ptr"] = K0.row_ptr
    out["K_col_idx"] = K0.col_idx
    out["K_values"] = np.stack([K.values for K in Ks])
    out["rhs"] = np.stack(rhss)
    f, d0 = R_lu.factorize(R_sc.to_general(K0))
    for k, v in factor_arrays(f).items():
        out[f"f0_{k}"] = v
    out["f0_diag"] = diag_vec(d0)
    keep = keep_factor_vals if keep_factor_vals is not None else range(len(Ks))
    x0s, spx, diags = [], [], []
    for i, (K, r) in enumerate(zip(Ks, rhss)):
        d = R_lu.refactorize(f, R_sc.to_general(K))
        diags.append(diag_vec(d))
        if i in keep:
            out[f"s{i}_Lx"] = f._Lx.copy()
            out[f"s{i}_Ux"] = f._Ux.copy()
            out[f"s{i}_Udiag"] = f._Udiag.copy()
        x0 = R_lu.lu_solve(f, r)
        x0s.append(x0)
        spx.append(R_sc.spmv(K, x0))
    out["refactor_diag"] = np.stack(diags)
    out["x0"] = np.stack(x0s)
    out["spmv_K_x0"] = np.stack(spx)
    for delta in deltas:
        tag = f"{delta:.0e}"
        xs, reps = [], []
        for i, (K, r) in enumerate(zip(Ks, rhss)):
            R_lu.refactorize(f, R_sc.to_general(K))
            x0 = R_lu.lu_solve(f, r)
            x, rep = refine_fgmres(K, f, x0, r, RefinementConfig(delta_tol=delta,
                                                                 krylov=KrylovConfig(m=10)))
            xs.append(x)
            reps.append([rep.triggered, rep.ir_iterations, rep.triangular_solves_used,
                         rep.nsr_before, rep.nsr_after, rep.rr_final, rep.nrbe_final,
                         rep.converged])
        out[f"refine_{tag}_x"] = np.stack(xs)
        out[f"refine_{tag}_report"] = np.array(reps, dtype=np.float64)
        seq = MatrixSequence(name, [SequenceItem(K=K, rhs=r) for K, r in zip(Ks, rhss)], {})
        rows = run_strategy(seq, StrategySpec("refactor_ir_fgmres", RefinementConfig(
            delta_tol=delta, krylov=KrylovConfig(m=10)))).rows
        out[f"harness_{tag}"] = np.array([[r.nsr_before, r.nsr_after, r.nrbe, r.rr,
                                           r.ir_iterations, r.triangular_solves]
                                          for r in rows])
    # Richardson IR (refine.py:135-205): tolerance stop at two deltas, NSR-ratio stop
    for tag, rcfg in (("1e-10", dict(delta_tol=1e-10)), ("1e-14", dict(delta_tol=1e-14)),
                      ("nsr", dict(delta_tol=1e-10, richardson_stop="nsr_ratio"))):
        xs, reps = [], []
        for i, (K, r) in enumerate(zip(Ks, rhss)):
            R_lu.refactorize(f, R_sc.to_general(K))
            x0 = R_lu.lu_solve(f, r)
            x, rep = refine_richardson(K, f, x0, r, RefinementConfig(**rcfg))
            xs.append(x)
            reps.append([rep.triggered, rep.ir_iterations, rep.triangular_solves_used,
                         rep.nsr_before, rep.nsr_after, rep.rr_final, rep.nrbe_final,
                         rep.converged, rep.diverged])
        out[f"richardson_{tag}_x"] = np.stack(xs)
        out[f"richardson_{tag}_report"] = np.array(reps, dtype=np.float64)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "N", K0.n_rows, "nnzL", f._Li.size, "iters",
          out["refine_1e-10_report"][:, 1].astype(int).tolist())


def standard():
    tr = standard_trace()
    Ks = [ks.K for ks, _r, _mu, _c in tr.systems]
    rhss = [np.concatenate([r.r_x, r.r_lambda]) for _k, r, _mu, _c in tr.systems]
    sequence_case("standard_trace", Ks, rhss, keep_factor_vals=[0, 4, 8])


def acopf_case(name, nbus, M):
    seq = acopf.make_sequence(nbus, seed=0, length=M)
    P = seq.pattern.K
    Ks = [R_sc.CsMatrix(P.n_rows, P.n_cols, P.row_ptr, P.col_idx, seq.values(k),
                        R_sc.SYMMETRIC_LOWER) for k in range(M)]
    rhss = [seq.rhs(k) for k in range(M)]
    sequence_case(name, Ks, rhss, keep_factor_vals=[0, M // 2, M - 1])


def random_cases():
    """conftest.random_sparse matrices: factorize + solve + refactorize(2A) (bitwise)."""
    out = {}
    rng = np.random.default_rng(2024)
    sizes = []
    for s in range(12):
        n = int(rng.integers(10, 160))
        A = random_sparse(n, 0.06, 5000 + s)
        f, d = R_lu.factorize(A)
        b = rng.standard_normal(n)
        x = R_lu.lu_solve(f, b)
        out[f"r{s}_row_ptr"] = A.row_ptr
        out[f"r{s}_col_idx"] = A.col_idx
        out[f"r{s}_values"] = A.values
        for k, v in factor_arrays(f).items():
            out[f"r{s}_{k}"] = v
        out[f"r{s}_diag"] = diag_vec(d)
        out[f"r{s}_b"] = b
        out[f"r{s}_x"] = x
        out[f"r{s}_spmv_b"] = R_sc.spmv(A, b)
        d2 = R_lu.refactorize(f, A.with_values(2.0 * A.values))
        out[f"r{s}_x2"] = R_lu.lu_solve(f, b)
        out[f"r{s}_Lx2"] = f._Lx.copy()
        out[f"r{s}_Ux2"] = f._Ux.copy()
        out[f"r{s}_Udiag2"] = f._Udiag.copy()
        out[f"r{s}_diag2"] = diag_vec(d2)
        sizes.append(n)
    out["count"] = np.array([12])
    np.savez_compressed(os.path.join(HERE, "random_sparse.npz"), **out)
    print("random_sparse sizes", sizes)


def edge_cases():
    out = {}
    # zero pivot patched (test_direct_lu.py:149-156 analogue)
    A = R_sc.from_dense(np.array([[2.0, 1.0], [1.0, 2.0]]))
    f, _ = R_lu.factorize(A)
    B = R_sc.from_dense(np.array([[2.0, 1.0], [1.0, 0.5]]))
    d = R_lu.refactorize(f, B)
    out["patch_A"] = A.values
    out["patch_B"] = B.values
    out["patch_diag"] = diag_vec(d)
    out["patch_Udiag"] = f._Udiag.copy()
    out["patch_Lx"] = f._Lx.copy()
    out["patch_x"] = R_lu.lu_solve(f, np.array([1.0, -1.0]))
    # forced swap
    S = R_sc.from_dense(np.array([[0.0, 1.0], [1.0, 0.0]]))
    g, _ = R_lu.factorize(S)
    out["swap_row_perm"] = g.row_perm.perm
    out["swap_col_perm"] = g.col_perm.perm
    np.savez_compressed(os.path.join(HERE, "edge_cases.npz"), **out)


def kkt_case():
    """Reference kkt.py (assemble_kkt / assemble_rhs / recover_dz) on the standard trace."""
    from kktsolve.kkt import assemble_kkt, assemble_rhs, recover_dz
    from kktsolve.seqgen import qp_residuals
    tr = standard_trace()
    out = {}
    ks0 = tr.systems[0][0]
    H, J = ks0.blocks.H, ks0.blocks.J
    out.update(H_row_ptr=H.row_ptr, H_col_idx=H.col_idx, H_values=H.values, J_row_ptr=J.row_ptr,
               J_col_idx=J.col_idx, J_values=J.values, n=np.array([H.n_rows, J.n_rows]))
    rng = np.random.default_rng(7)
    xs, zs, mus, Kv, Kd, rts, rls, rzs, rxs, dxs, dzs = ([] for _ in range(11))
    donor = None
    for ks, rhs, mu, _c in tr.systems:
        b = ks.blocks
        k2 = assemble_kkt(b, pattern_from=donor)
        if donor is None:
            k_fresh = assemble_kkt(b)
            assert np.array_equal(k_fresh.K.values, k2.K.values)
        donor = k2
        rt = rhs.r_tilde_x
        r2 = assemble_rhs(b, rt, rhs.r_lambda, rhs.r_z)
        dx = rng.standard_normal(b.n)
        xs.append(b.x); zs.append(b.z); mus.append(b.mu); Kv.append(k2.K.values)
        Kd.append(k2.dx_diag); rts.append(rt); rls.append(rhs.r_lambda); rzs.append(rhs.r_z)
        rxs.append(r2.r_x); dxs.append(dx); dzs.append(recover_dz(b, rhs.r_z, dx))
    out.update(K_row_ptr=donor.K.row_ptr, K_col_idx=donor.K.col_idx, x=np.stack(xs), z=np.stack(zs),
               mu=np.array(mus), K_values=np.stack(Kv), dx_diag=np.stack(Kd), r_tilde_x=np.stack(rts),
               r_lambda=np.stack(rls), r_z=np.stack(rzs), r_x=np.stack(rxs), dx=np.stack(dxs),
               dz=np.stack(dzs))
    np.savez_compressed(os.path.join(HERE, "kkt_assembly.npz"), **out)
    print("kkt_assembly", len(xs), "systems, nnz(K)", donor.K.nnz)


def mm_case():
    """Reference mmio on files written by the reference: parsed arrays + error messages."""
    from kktsolve import mmio as R_mm
    d = os.path.join(HERE, "mm")
    os.makedirs(d, exist_ok=True)
    tr = standard_trace()
    K = tr.systems[3][0].K
    R_mm.write_matrix_market(os.path.join(d, "K_sym.mtx"), K)
    R_mm.write_matrix_market(os.path.join(d, "K_gen.mtx"), R_sc.to_general(K))
    R_mm.write_vector(os.path.join(d, "r.mtx"), tr.systems[3][1].r_x)
    bad = {
        "bad_header.mtx": "%%MatrixMarket vector coordinate real general\n1 1 1\n1 1 1.0\n",
        "bad_field.mtx": "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1.0\n",
        "bad_size.mtx": "%%MatrixMarket matrix coordinate real general\n% c\n2 2\n",
        "bad_entry.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n2 x 3.0\n",
        "bad_range.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
        "bad_upper.mtx": "%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 2 1.0\n",
        "bad_count.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n",
        "bad_extra.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n2 2 2.0\n",
    }
    msgs = {}
    for name, text in bad.items():
        path = os.path.join(d, name)
        with open(path, "w") as fh:
            fh.write(text)
        try:
            R_mm.load_matrix_market(path)
            msgs[name] = None
        except R_mm.MatrixMarketError as exc:
            msgs[name] = str(exc).replace(d, "<dir>")
    out = {}
    for name in ("K_sym.mtx", "K_gen.mtx"):
        A = R_mm.load_matrix_market(os.path.join(d, name))
        tag = name.split(".")[0]
        out[f"{tag}_row_ptr"], out[f"{tag}_col_idx"], out[f"{tag}_values"] = A.row_ptr, A.col_idx, A.values
        out[f"{tag}_sym"] = np.array([A.symmetry == R_sc.SYMMETRIC_LOWER])
    out["r"] = R_mm.load_vector(os.path.join(d, "r.mtx"))
    np.savez_compressed(os.path.join(d, "expected.npz"), **out)
    with open(os.path.join(d, "errors.json"), "w") as fh:
        json.dump(msgs, fh, indent=1)
    print("mm files", sorted(msgs))


def main():
    meta = {"reference": "/root/reference/pkg (kktsolve 0.1.0)", "numpy": np.__version__}
    standard()
    acopf_case("acopf_tiny", acopf.ACOPF_CONFIGS["tiny"], 20)
    acopf_case("acopf_small", acopf.ACOPF_CONFIGS["small"], 20)
    random_cases()
    edge_cases()
    kkt_case()
    mm_case()
    with open(os.path.join(HERE, "MANIFEST.json"), "w") as fh:
        json.dump(meta, fh, indent=2)


if __name__ == "__main__":
    main()
