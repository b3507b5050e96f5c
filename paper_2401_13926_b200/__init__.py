"""B200-native KKT refactorization + FGMRES-IR hot path (arXiv:2401.13926).

Drop-in for the hot-path API of the reference package ``kktsolve`` (its ``__init__.py``
re-exports, pkg/src/kktsolve/__init__.py:17-71, restricted to the refactor/solve/refine
path): ``factorize`` (host analysis, C++), ``refactorize`` / ``lu_solve`` / ``spmv`` /
``fgmres`` / ``refine_fgmres`` (sm_100a kernels behind ``libkktb200.so``).
"""

from .sparse import (GENERAL, SYMMETRIC_LOWER, CsMatrix, Permutation, SparseError, Triplets,
                     from_dense, from_triplets, identity, to_general)
from .direct_lu import (PATCH_RELATIVE_FLOOR, LuDiagnostics, LuFactors, PatternMismatchError,
                        SingularMatrixError, factorize, lu_solve, refactorize)
from .krylov import (CGS2, MGS, KrylovConfig, KrylovResult, LinearOperator, NotSpdOperatorError,
                     OperatorOutputError, fgmres, lu_preconditioner)
from .refine import (BarrierTiedTolerance, FixedTolerance, RefinementConfig, RefinementReport,
                     config_for_mu, needs_refinement, nrbe, nsr, refine_fgmres,
                     refine_richardson)
from .sparse_ops import inf_norm, spmv
from .kkt import (DeviceKktAssembler, KktBlocks, KktRhs, KktSystem, assemble_kkt, assemble_rhs,
                  recover_dz)

__all__ = [name for name in dir() if not name.startswith("_")]
__version__ = "0.1.0"
