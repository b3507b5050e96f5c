"""Shared test plumbing.  `-m gpu` tests need a CUDA device (the B200 box); everything else
runs on the CPU build container."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session", autouse=True)
def _built_library():
    from paper_2401_13926_b200 import build
    build.build()
    yield


def golden(name: str):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def lower_matrix(g, k: int):
    from paper_2401_13926_b200.sparse import SYMMETRIC_LOWER, CsMatrix
    n = int(g["n"][0])
    return CsMatrix(n, n, g["K_row_ptr"], g["K_col_idx"], g["K_values"][k].copy(),
                    SYMMETRIC_LOWER)


FACTOR_KEYS = ["row_perm", "col_perm", "Lp", "Li", "Lx", "Up", "Ui", "Ux", "Udiag", "so_ptr",
               "so_data", "ap_ptr", "a_src", "a_tgt"]


def factor_dict(f) -> dict:
    return dict(row_perm=f.row_perm.perm, col_perm=f.col_perm.perm, Lp=f._Lp, Li=f._Li,
                Lx=f._Lx, Up=f._Up, Ui=f._Ui, Ux=f._Ux, Udiag=f._Udiag, so_ptr=f._so_ptr,
                so_data=f._so_data, ap_ptr=f._ap_ptr, a_src=f._a_src, a_tgt=f._a_tgt)
