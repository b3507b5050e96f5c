"""Matrix Market ingestion in C++ (mmio.py:36-155) against the
reference: files written by the reference's writer parse to the reference's arrays
(bitwise), our writer round-trips exactly, and malformed files raise MatrixMarketError
with the reference's "path:line: message" (ours is a prefix of the reference's, which
appends Python's exception text)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2401_13926_b200.mmio import (MatrixMarketError, load_matrix_market, load_vector,
                                        write_matrix_market, write_vector)
from paper_2401_13926_b200.sparse import SYMMETRIC_LOWER

D = os.path.join(GOLDEN, "mm")


@pytest.mark.parametrize("tag", ["K_sym", "K_gen"])
def test_reference_files_parse_bitwise(tag):
    e = np.load(os.path.join(D, "expected.npz"))
    A = load_matrix_market(os.path.join(D, f"{tag}.mtx"))
    assert np.array_equal(A.row_ptr, e[f"{tag}_row_ptr"])
    assert np.array_equal(A.col_idx, e[f"{tag}_col_idx"])
    assert np.array_equal(A.values, e[f"{tag}_values"])
    assert (A.symmetry == SYMMETRIC_LOWER) == bool(e[f"{tag}_sym"][0])


def test_vector_and_round_trip(tmp_path):
    e = np.load(os.path.join(D, "expected.npz"))
    r = load_vector(os.path.join(D, "r.mtx"))
    assert np.array_equal(r, e["r"])
    A = load_matrix_market(os.path.join(D, "K_sym.mtx"))
    write_matrix_market(tmp_path / "a.mtx", A)
    write_vector(tmp_path / "v.mtx", r)
    B = load_matrix_market(tmp_path / "a.mtx")
    assert np.array_equal(A.values, B.values) and np.array_equal(A.col_idx, B.col_idx)
    assert np.array_equal(load_vector(tmp_path / "v.mtx"), r)


def test_errors_match_reference():
    msgs = json.load(open(os.path.join(D, "errors.json")))
    for name, ref in msgs.items():
        with pytest.raises(MatrixMarketError) as ei:
            load_matrix_market(os.path.join(D, name))
        ours = str(ei.value).replace(D, "<dir>")
        assert ref.startswith(ours), (name, ours, ref)


def test_load_sequence_manifest(tmp_path):
    """harness.load_sequence over files in the reference's export layout."""
    import shutil
    from paper_2401_13926_b200.harness import SequenceError, load_sequence
    n = load_matrix_market(os.path.join(D, "K_sym.mtx")).n_rows
    for i in range(2):
        shutil.copy(os.path.join(D, "K_sym.mtx"), tmp_path / f"s_K{i:03d}.mtx")
        write_vector(tmp_path / f"s_rhs{i:03d}.mtx", np.arange(n, dtype=float) / 3.0)
    man = {"name": "s", "systems": [{"matrix": f"s_K{i:03d}.mtx", "rhs": f"s_rhs{i:03d}.mtx"}
                                    for i in range(2)], "n": 200, "m": 50, "mu": [1.0, 0.1]}
    (tmp_path / "m.json").write_text(json.dumps(man))
    seq = load_sequence(str(tmp_path / "m.json"))
    assert len(seq.items) == 2 and seq.metadata["mu"] == [1.0, 0.1]
    assert seq.metadata["N"] == seq.items[0].K.n_rows
    shutil.copy(os.path.join(D, "K_gen.mtx"), tmp_path / "s_K001.mtx")
    with pytest.raises(SequenceError):
        load_sequence(str(tmp_path / "m.json"))
