"""KKT assembly / rhs reduction / dz recovery (kkt.py:88-144) against
the reference's outputs on its standard barrier trace (tests/golden/kkt_assembly.npz).

CPU: the frozen pattern and the scatter maps (integer plumbing).  GPU: every value —
K (fresh and pattern-reusing), D_x, r_x, dz — bitwise, single-system drop-in and batched."""

import numpy as np
import pytest

from conftest import golden
from paper_2401_13926_b200.kkt import KktBlocks, _row_of_entry, entry_positions, source_map
from paper_2401_13926_b200.sparse import GENERAL, SYMMETRIC_LOWER, CsMatrix, Triplets, from_triplets


def _blocks(g, i):
    n, m = (int(v) for v in g["n"])
    H = CsMatrix(n, n, g["H_row_ptr"], g["H_col_idx"], g["H_values"].copy(), SYMMETRIC_LOWER)
    J = CsMatrix(m, n, g["J_row_ptr"], g["J_col_idx"], g["J_values"].copy(), GENERAL)
    return KktBlocks(H=H, J=J, x=g["x"][i], z=g["z"][i], mu=float(g["mu"][i]))


def test_pattern_and_maps_match_reference():
    g = golden("kkt_assembly")
    b = _blocks(g, 0)
    n, m = b.n, b.m
    rows = np.concatenate([_row_of_entry(b.H), np.arange(n), _row_of_entry(b.J) + n])
    cols = np.concatenate([b.H.col_idx, np.arange(n), b.J.col_idx])
    K = from_triplets(Triplets(n + m, n + m, rows, cols, np.zeros(rows.size)), SYMMETRIC_LOWER)
    assert np.array_equal(K.row_ptr, g["K_row_ptr"]) and np.array_equal(K.col_idx, g["K_col_idx"])
    h_pos = entry_positions(K, _row_of_entry(b.H), b.H.col_idx)
    d_pos = entry_positions(K, np.arange(n), np.arange(n))
    j_pos = entry_positions(K, _row_of_entry(b.J) + n, b.J.col_idx)
    src = source_map(K.nnz, n, h_pos, d_pos, j_pos)
    assert (src[:, 0] >= 0).all()  # every stored entry has a source
    # numpy restatement of the reference's np.add.at scatter, using the map, on system 0
    vals = np.zeros(K.nnz)
    srcv = np.concatenate([b.H.values, b.z / b.x, b.J.values])
    vals += srcv[src[:, 0]]
    two = src[:, 1] >= 0
    vals[two] = vals[two] + srcv[src[two, 1]]
    assert np.array_equal(vals, g["K_values"][0])


@pytest.mark.gpu
def test_device_assembly_bitwise_dropin():
    from paper_2401_13926_b200.kkt import assemble_kkt, assemble_rhs, recover_dz
    g = golden("kkt_assembly")
    donor = None
    for i in range(g["x"].shape[0]):
        b = _blocks(g, i)
        ks = assemble_kkt(b, pattern_from=donor)
        if donor is None:
            assert np.array_equal(ks.K.row_ptr, g["K_row_ptr"])
        donor = ks
        assert np.array_equal(ks.K.values, g["K_values"][i]), i
        assert np.array_equal(ks.dx_diag, g["dx_diag"][i]), i
        r = assemble_rhs(b, g["r_tilde_x"][i], g["r_lambda"][i], g["r_z"][i])
        assert np.array_equal(r.r_x, g["r_x"][i]), i
        assert np.array_equal(recover_dz(b, g["r_z"][i], g["dx"][i]), g["dz"][i]), i


@pytest.mark.gpu
def test_device_assembly_batched():
    import torch
    from paper_2401_13926_b200.kkt import DeviceKktAssembler, assemble_kkt
    g = golden("kkt_assembly")
    M = g["x"].shape[0]
    ks = assemble_kkt(_blocks(g, 0))
    asm = DeviceKktAssembler(ks, nb=M)
    n, m = ks.n, ks.m
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(asm.device)  # noqa: E731
    with torch.cuda.stream(asm.stream):
        H = dev(np.tile(g["H_values"], (M, 1)))
        J = dev(np.tile(g["J_values"], (M, 1)))
        x, z, mu = dev(g["x"]), dev(g["z"]), dev(g["mu"])
        K = torch.empty((M, ks.K.nnz), dtype=torch.float64, device=asm.device)
        rhs = torch.empty((M, n + m), dtype=torch.float64, device=asm.device)
        sol = dev(np.concatenate([g["dx"], np.zeros((M, m))], 1))
        dz = torch.empty((M, n), dtype=torch.float64, device=asm.device)
    asm.values(H, J, x, z, K)
    asm.rhs(dev(g["r_tilde_x"]), dev(g["r_lambda"]), x, z, mu, rhs)
    asm.recover_dz(dev(g["r_z"]), z, sol, x, dz, dx_stride=n + m)
    asm.stream.synchronize()
    assert np.array_equal(K.cpu().numpy(), g["K_values"])
    r = rhs.cpu().numpy()
    assert np.array_equal(r[:, :n], g["r_x"]) and np.array_equal(r[:, n:], g["r_lambda"])
    assert np.array_equal(dz.cpu().numpy(), g["dz"])
