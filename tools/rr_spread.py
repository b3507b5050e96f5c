"""How reproducible is the reference's final residual under a different summation order?

For every refined system of the BASELINE-size reference goldens (tests/golden/large_*.npz,
written by the REFERENCE itself), run the plain-C oracle (oracle/kkt_oracle.c: the same
algorithm, sequential dot products instead of OpenBLAS ddot/dgemv) on the same inputs and
print the reference's true rr, the oracle's, their ratio and both iteration counts.
The spread bounds the residual parity bar (tests/large_golden.rr_bound).

    python tools/rr_spread.py [case ...]      (build container: needs the goldens only)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from large_golden import CASES, M, REPORT, available, barrier_delta, load, sequence  # noqa: E402


def main(cases):
    import bench
    from oracle import oracle
    from paper_2401_13926_b200 import factorize, to_general
    worst_eq = 0.0
    for case in cases:
        g, seq = load(case), sequence(case)
        K0 = seq.matrix(0)
        f, _ = factorize(to_general(K0))
        of, ex = bench.oracle_factors(f, K0)
        for tag in ("1e-10", "barrier"):
            for k in range(M):
                r = dict(zip(REPORT, g[f"refine_{tag}"][k]))
                if not r["triggered"]:
                    continue
                v, rhs, K = seq.values(k), seq.rhs(k), seq.matrix(k)
                d = 1e-10 if tag == "1e-10" else barrier_delta(seq, k)
                of.refactorize(v[ex.src])
                x, rep = of.refine_fgmres(K.row_ptr, K.col_idx, v, rhs, of.lu_solve(rhs), d)
                rr = np.linalg.norm(rhs - oracle.spmv(K.row_ptr, K.col_idx, v, x)) / np.linalg.norm(rhs)
                ratio = rr / r["rr_true"]
                same = rep["iterations"] == int(r["ir_iterations"])
                if same:
                    worst_eq = max(worst_eq, ratio)
                print(f"{case:13s} {tag:8s} k={k:2d} it ref {int(r['ir_iterations']):2d} oracle "
                      f"{rep['iterations']:2d}  rr ref {r['rr_true']:.2e} oracle {rr:.2e} "
                      f"ratio {ratio:6.2f}  delta {d:.0e}", flush=True)
    print(f"worst oracle/reference rr ratio at equal iteration counts: {worst_eq:.2f}")


if __name__ == "__main__":
    main([c for c in (sys.argv[1:] or CASES) if available(c)])
