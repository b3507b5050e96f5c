"""Drop-in for ``kktsolve.kkt``: assembly of the reduced saddle-point systems of an
interior-point iteration, with the floating-point work on the B200.

``assemble_kkt`` freezes the combined pattern ``[[H + D_x, J^T], [J, 0]]`` once (host,
integer plumbing, kkt.py:88-124) and every value — H and J scattered, ``D_x = z / x`` added
on the diagonal in np.add.at order — is produced by ``kkt_assemble_values`` on the device.
``assemble_rhs`` (kkt.py:127-137) and ``recover_dz`` (kkt.py:140-144) likewise run as device
kernels.  :class:`DeviceKktAssembler` is the batched, device-resident form: values, rhs and
dz of ``nb`` systems from device arrays, feeding ``DeviceSystem.step`` without host traffic.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .sparse import SYMMETRIC_LOWER, CsMatrix, SparseError, Triplets, from_triplets


@dataclass
class KktBlocks:
    """Blocks of one saddle-point system at a strictly interior point (kkt.py:27-54)."""

    H: CsMatrix
    J: CsMatrix
    x: np.ndarray
    z: np.ndarray
    mu: float

    def __post_init__(self):
        self.x = np.asarray(self.x, dtype=np.float64)
        self.z = np.asarray(self.z, dtype=np.float64)
        n = self.H.n_rows
        if self.H.symmetry != SYMMETRIC_LOWER:
            raise SparseError("H must use symmetric-lower storage")
        if self.J.n_cols != n or self.x.shape != (n,) or self.z.shape != (n,):
            raise SparseError("KKT block dimensions do not conform")
        if np.any(self.x <= 0.0) or np.any(self.z <= 0.0):
            raise ValueError("interior point violated: x and z must be positive")

    @property
    def n(self) -> int:
        return self.H.n_rows

    @property
    def m(self) -> int:
        return self.J.n_rows


class KktSystem:
    """The assembled ``(n+m) x (n+m)`` matrix plus its frozen scatter maps (kkt.py:57-79)."""

    def __init__(self, K: CsMatrix, blocks: KktBlocks, dx_diag, h_pos, d_pos, j_pos, src=None):
        self.K = K
        self.blocks = blocks
        self.dx_diag = dx_diag
        self._h_pos = h_pos
        self._d_pos = d_pos
        self._j_pos = j_pos
        self._src = src if src is not None else source_map(K.nnz, blocks.n, h_pos, d_pos, j_pos)

    @property
    def n(self) -> int:
        return self.blocks.n

    @property
    def m(self) -> int:
        return self.blocks.m


@dataclass
class KktRhs:
    r_x: np.ndarray
    r_lambda: np.ndarray
    r_z: np.ndarray
    r_tilde_x: np.ndarray


def _row_of_entry(A: CsMatrix) -> np.ndarray:
    return np.repeat(np.arange(A.n_rows, dtype=np.int64), np.diff(A.row_ptr))


def entry_positions(K: CsMatrix, rows, cols) -> np.ndarray:
    """Positions of (row, col) pairs in K's storage (sparsecore.entry_positions, :472)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    key_k = _row_of_entry(K) * K.n_cols + K.col_idx   # sorted: rows ascending, cols sorted
    key = rows * K.n_cols + cols
    pos = np.searchsorted(key_k, key)
    if np.any(pos >= key_k.size) or np.any(key_k[np.minimum(pos, key_k.size - 1)] != key):
        raise SparseError("entry absent from target pattern")
    return pos.astype(np.int64)


def source_map(nnz: int, n: int, h_pos, d_pos, j_pos) -> np.ndarray:
    """[nnz][2] int32: the ordered sources of every K position (H, then D, then J)."""
    nH = h_pos.size
    src = np.full((nnz, 2), -1, dtype=np.int32)
    for ids, pos in ((np.arange(nH), h_pos), (nH + np.arange(n), d_pos),
                     (nH + n + np.arange(j_pos.size), j_pos)):
        slot = (src[pos, 0] >= 0).astype(np.int64)
        if np.any(src[pos[slot == 1], 1] >= 0):
            raise SparseError("more than two sources for one KKT entry")
        src[pos, slot] = ids
    return src


class DeviceKktAssembler:
    """Device-resident assembly for ``nb`` systems sharing one frozen KKT pattern."""

    def __init__(self, ksys: KktSystem, nb: int = 1, device: int = 0):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("kktb200: no CUDA device visible (no CPU fallback)")
        self.torch = torch
        self.lib = nat.load()
        self.device = torch.device("cuda", device)
        self.stream = torch.cuda.Stream(device=self.device)
        self.nb = int(nb)
        self.n, self.m = ksys.n, ksys.m
        self.nH, self.nJ = ksys.blocks.H.nnz, ksys.blocks.J.nnz
        self.nnz = ksys.K.nnz
        with torch.cuda.stream(self.stream):
            self.src = torch.from_numpy(np.ascontiguousarray(ksys._src)).to(self.device)
        self.stream.synchronize()

    def _ptr(self, t):
        return C.c_void_p(t.data_ptr()) if t is not None else None

    def values(self, H_t, J_t, x_t, z_t, K_t):
        """K_t[nb][nnz] <- the assembled symmetric-lower values (kkt.py:104-107)."""
        nat.check(self.lib.kkt_assemble_values(self.nnz, self.n, self.nH, self.nJ, self.nb,
                                               self._ptr(self.src), self._ptr(H_t), self._ptr(J_t),
                                               self._ptr(x_t), self._ptr(z_t), self._ptr(K_t),
                                               C.c_void_p(self.stream.cuda_stream)),
                  "kkt_assemble_values")

    def rhs(self, rtx_t, rl_t, x_t, z_t, mu_t, rhs_t):
        """rhs_t[nb][n+m] <- [r~_x + (z - mu/x); r_lambda] (kkt.py:136)."""
        nat.check(self.lib.kkt_assemble_rhs(self.n, self.m, self.nb, self._ptr(rtx_t), self._ptr(rl_t),
                                            self._ptr(x_t), self._ptr(z_t), self._ptr(mu_t),
                                            self._ptr(rhs_t), C.c_void_p(self.stream.cuda_stream)),
                  "kkt_assemble_rhs")

    def recover_dz(self, rz_t, z_t, dx_t, x_t, dz_t, dx_stride: int | None = None):
        """dz_t[nb][n] <- (r_z - z dx)/x (kkt.py:144); dx rows are dx_stride apart."""
        nat.check(self.lib.kkt_recover_dz(self.n, self.nb, int(dx_stride or self.n), self._ptr(rz_t),
                                          self._ptr(z_t), self._ptr(dx_t), self._ptr(x_t),
                                          self._ptr(dz_t), C.c_void_p(self.stream.cuda_stream)),
                  "kkt_recover_dz")


def _dev(t, a):
    return t.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def assemble_kkt(blocks: KktBlocks, pattern_from: KktSystem | None = None) -> KktSystem:
    """Assemble the reduced system; reuse a previous system's frozen pattern (kkt.py:88)."""
    n, m = blocks.n, blocks.m
    if pattern_from is not None:
        prev = pattern_from
        if not (blocks.H.same_pattern(prev.blocks.H) and blocks.J.same_pattern(prev.blocks.J)):
            raise SparseError("assemble_kkt: block patterns differ from the pattern-donor system")
        K0, h_pos, d_pos, j_pos, src = prev.K, prev._h_pos, prev._d_pos, prev._j_pos, prev._src
    else:
        h_rows = _row_of_entry(blocks.H)
        j_rows = _row_of_entry(blocks.J) + n
        d_idx = np.arange(n, dtype=np.int64)
        rows = np.concatenate([h_rows, d_idx, j_rows])
        cols = np.concatenate([blocks.H.col_idx, d_idx, blocks.J.col_idx])
        K0 = from_triplets(Triplets(n + m, n + m, rows, cols, np.zeros(rows.size)), SYMMETRIC_LOWER)
        h_pos = entry_positions(K0, h_rows, blocks.H.col_idx)
        d_pos = entry_positions(K0, d_idx, d_idx)
        j_pos = entry_positions(K0, j_rows, blocks.J.col_idx)
        src = source_map(K0.nnz, n, h_pos, d_pos, j_pos)
    import torch
    ksys = KktSystem(K0, blocks, None, h_pos, d_pos, j_pos, src)
    asm = DeviceKktAssembler(ksys)
    with torch.cuda.stream(asm.stream):
        Ht, Jt = _dev(torch, blocks.H.values), _dev(torch, blocks.J.values)
        xt, zt = _dev(torch, blocks.x), _dev(torch, blocks.z)
        Kt = torch.empty(K0.nnz, dtype=torch.float64, device=asm.device)
    asm.values(Ht, Jt, xt, zt, Kt)
    # D_x = z / x itself (KktSystem.dx_diag): the same kernel with D as the only source
    lib = nat.load()
    with torch.cuda.stream(asm.stream):
        src_d = torch.from_numpy(np.stack([blocks.H.nnz + np.arange(n, dtype=np.int32),
                                           np.full(n, -1, dtype=np.int32)], 1).copy()).to(asm.device)
        Dt = torch.empty(n, dtype=torch.float64, device=asm.device)
    nat.check(lib.kkt_assemble_values(n, n, blocks.H.nnz, blocks.J.nnz, 1, C.c_void_p(src_d.data_ptr()),
                                      C.c_void_p(Ht.data_ptr()), C.c_void_p(Jt.data_ptr()),
                                      C.c_void_p(xt.data_ptr()), C.c_void_p(zt.data_ptr()),
                                      C.c_void_p(Dt.data_ptr()), C.c_void_p(asm.stream.cuda_stream)),
              "kkt_assemble_values")
    with torch.cuda.stream(asm.stream):
        vals = Kt.cpu().numpy()
        ksys.dx_diag = Dt.cpu().numpy()
    ksys.K = K0.with_values(vals)
    return ksys


def assemble_rhs(blocks: KktBlocks, r_tilde_x, r_lambda, r_z) -> KktRhs:
    """``r_x = r~_x + (z - mu X^-1 e)`` on the device (kkt.py:127-137)."""
    import torch
    r_tilde_x = np.asarray(r_tilde_x, dtype=np.float64)
    r_lambda = np.asarray(r_lambda, dtype=np.float64)
    r_z = np.asarray(r_z, dtype=np.float64)
    if r_tilde_x.shape != (blocks.n,) or r_lambda.shape != (blocks.m,) or r_z.shape != (blocks.n,):
        raise ValueError("assemble_rhs: length mismatch")
    lib = nat.load()
    rhs = torch.empty(blocks.n + blocks.m, dtype=torch.float64, device="cuda")
    args = [_dev(torch, a) for a in (r_tilde_x, r_lambda, blocks.x, blocks.z, [blocks.mu])]
    nat.check(lib.kkt_assemble_rhs(blocks.n, blocks.m, 1, *[C.c_void_p(t.data_ptr()) for t in args],
                                   C.c_void_p(rhs.data_ptr()), None), "kkt_assemble_rhs")
    r_x = rhs[:blocks.n].cpu().numpy()
    return KktRhs(r_x=r_x, r_lambda=r_lambda, r_z=r_z, r_tilde_x=r_tilde_x)


def recover_dz(blocks: KktBlocks, r_z, dx) -> np.ndarray:
    """Bound-multiplier step from ``X dz = r_z - Z dx`` on the device (kkt.py:140-144)."""
    import torch
    lib = nat.load()
    args = [_dev(torch, a) for a in (r_z, blocks.z, dx, blocks.x)]
    dz = torch.empty(blocks.n, dtype=torch.float64, device="cuda")
    nat.check(lib.kkt_recover_dz(blocks.n, 1, blocks.n, *[C.c_void_p(t.data_ptr()) for t in args],
                                 C.c_void_p(dz.data_ptr()), None), "kkt_recover_dz")
    return dz.cpu().numpy()
