"""The C-ABI library loads and exports every symbol include/kktb200.h declares (CPU-only)."""

import ctypes as C
import os
import re

from conftest import ROOT
from paper_2401_13926_b200 import _native as nat


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "kktb200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kkt_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported_and_typed():
    lib = nat.load()
    names = declared_symbols()
    assert len(names) >= 25
    typed = {n for n, _, _ in nat.SIGNATURES}
    for name in names:
        assert hasattr(lib, name), name
        assert name in typed, f"{name} missing from _native.SIGNATURES"


def test_abi_version_and_error_string():
    lib = nat.load()
    assert lib.kkt_abi_version() == nat.ABI_VERSION
    h = C.c_void_p()
    rc = lib.kkt_analyze(2, None, None, None, 0.0, C.byref(h))
    assert rc == nat.KKT_ERR_BAD_ARG
    assert "pivot_tol" in nat.last_error()


def test_min_degree_export_matches_analysis():
    import numpy as np
    from conftest import golden, lower_matrix
    from paper_2401_13926_b200 import to_general
    g = golden("standard_trace")
    A = to_general(lower_matrix(g, 0))
    perm = np.empty(A.n_rows, dtype=np.int64)
    assert nat.load().kkt_min_degree_order(A.n_rows, nat.ptr_i64(A.row_ptr),
                                           nat.ptr_i64(A.col_idx), nat.ptr_i64(perm)) == 0
    assert np.array_equal(perm, g["f0_col_perm"])
