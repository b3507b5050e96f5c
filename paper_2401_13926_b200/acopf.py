"""Synthetic ACOPF-shaped KKT sequences (the benchmark and parity inputs).

The reference generator (``seqgen.barrier_sequence``, seqgen.py:135) cannot reach the
named sizes (its SpGEMM plan allocates a dense N x N accumulator, sparsecore.py:457, and
every Newton step runs a Python factorize, seqgen.py:182).  This module builds what
SURVEY.md §8(d) prescribes instead, deterministically from a seed:

* bus graph: near-planar (jittered grid, random spanning tree + extra local lines),
  lines ~= 1.27 * buses, ~25 % of buses carry a generator;
* primal block x: (Va, Vm) per bus, (Pg, Qg) per generator, one slack per flow-limit
  row, and a (P, Q) imbalance slack on a fraction of buses;
* H (lower): diagonal + (Va_i,Va_k), (Vm_i,Vm_k) line couplings + Va/Vm bus coupling;
* J: P/Q balance rows over the bus, its neighbours and its generators; two flow-limit
  rows per line (4 voltage entries + its slack);
* K = [[H + D_x, J^T], [J, 0]] in symmetric-lower storage, D_x = z / x;
* system 0 is well scaled (x = z = 1); system k has mu_k = 10^(-0.4k); bounded variables
  are active with a per-class probability: active x = mu^0.8*U(.5,2), z = U(.5,2); inactive
  x = U(.5,2), z = mu^0.8*U(.5,2) (free angles have no barrier term).  Calibrated with the
  oracle at N~238k: IR at delta=1e-10 triggers on 7/19 systems, 3.3 iterations on average,
  none exhausting max_outer (SURVEY.md §8d gates);
  H/J values jitter by +-1 % per step on the frozen pattern.

Shapes (``ACOPF_CONFIGS``) follow BASELINE.json: ~9k (ACTIVSg200-like CPU case), ~90k
(ACTIVSg2000), ~238k / nnz_lower ~0.7M (ACTIVSg10k), ~1.6M (ACTIVSg70k).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .sparse import SYMMETRIC_LOWER, CsMatrix

# name -> number of buses (N ~= 11.6 * buses with the default densities)
ACOPF_CONFIGS = {
    "tiny": 40,
    "small": 200,
    "activsg200": 780,       # N ~ 9k   (BASELINE configs[0], CPU-runnable)
    "activsg2000": 7800,     # N ~ 90k  (configs[1])
    "activsg10k": 20560,     # N ~ 238k (configs[2], the headline)
    "activsg70k": 141600,    # N ~ 1.64M (configs[3])
}


# Per-shape calibration of the D_x spread (active x = mu^d_exp * U(.5, 2)), checked with the
# oracle (tools/calibrate.py, SURVEY.md §8d gates).  0.8 everywhere except ACTIVSg70k, where
# 0.8 drives the last barrier step to 49-51 FGMRES iterations; 0.7 keeps k = 17..19 at 2
# (delta = 1e-10 triggers on 8/19 systems, 2 iterations each; profiles/r2_calibration_70k.txt).
ACOPF_D_EXP = {141600: 0.7}


@dataclass
class AcopfPattern:
    """Frozen structure of one ACOPF-shaped KKT family."""

    nbus: int
    n: int                      # primal variables
    m: int                      # constraint rows
    K: CsMatrix                 # symmetric-lower pattern (values of system 0)
    # triplet -> position map: K.values = sums of raw triplet values via `pos`
    pos: np.ndarray
    kind: np.ndarray            # 0 = H offdiag, 1 = H diag (+D), 2 = J
    var_of_diag: np.ndarray     # for kind==1 triplets: the x variable
    base: np.ndarray            # system-0 raw triplet values (H part without D)
    meta: dict = field(default_factory=dict)

    @property
    def N(self) -> int:
        return self.n + self.m


def _bus_graph(nbus: int, rng: np.random.Generator, extra_ratio: float = 0.27):
    R = int(np.ceil(np.sqrt(nbus)))
    idx = np.arange(nbus)
    r, c = idx // R, idx % R
    cand = []
    right = (c + 1 < R) & (idx + 1 < nbus)
    cand.append(np.stack([idx[right], idx[right] + 1], 1))
    down = idx + R < nbus
    cand.append(np.stack([idx[down], idx[down] + R], 1))
    diag = (c + 1 < R) & (idx + R + 1 < nbus)
    cand.append(np.stack([idx[diag], idx[diag] + R + 1], 1))
    E = np.concatenate(cand)
    E = E[rng.permutation(E.shape[0])]
    parent = np.arange(nbus)

    def find(a):
        root = a
        while parent[root] != root:
            root = parent[root]
        while parent[a] != root:
            parent[a], a = root, parent[a]
        return root

    tree, rest = [], []
    for e in range(E.shape[0]):
        a, b = find(E[e, 0]), find(E[e, 1])
        if a != b:
            parent[a] = b
            tree.append(e)
        else:
            rest.append(e)
    n_extra = min(len(rest), int(round(extra_ratio * nbus)))
    lines = E[np.array(tree + rest[:n_extra], dtype=np.int64)]
    lines = np.sort(lines, axis=1)
    return lines[np.lexsort((lines[:, 1], lines[:, 0]))]


def build_pattern(nbus: int, seed: int = 0, gen_frac: float = 0.25,
                  imbalance_frac: float = 1.0) -> AcopfPattern:
    rng = np.random.default_rng(seed)
    lines = _bus_graph(nbus, rng)
    L = lines.shape[0]
    gens = np.sort(rng.choice(nbus, size=max(1, int(round(gen_frac * nbus))), replace=False))
    G = gens.size
    imb = np.sort(rng.choice(nbus, size=int(round(imbalance_frac * nbus)), replace=False))
    S = imb.size
    # x-block layout
    va = np.arange(nbus)
    vm = nbus + np.arange(nbus)
    pg = 2 * nbus + np.arange(G)
    qg = 2 * nbus + G + np.arange(G)
    sf = 2 * nbus + 2 * G + np.arange(L)          # flow-from slacks
    st = 2 * nbus + 2 * G + L + np.arange(L)      # flow-to slacks
    sp = 2 * nbus + 2 * G + 2 * L + np.arange(S)  # P imbalance slacks
    sq = 2 * nbus + 2 * G + 2 * L + S + np.arange(S)
    n = 2 * nbus + 2 * G + 2 * L + 2 * S
    # constraint rows (absolute K row = n + row)
    rP = n + np.arange(nbus)
    rQ = n + nbus + np.arange(nbus)
    rF = n + 2 * nbus + np.arange(L)
    rT = n + 2 * nbus + L + np.arange(L)
    m = 2 * nbus + 2 * L
    N = n + m

    rows, cols, kind, vals = [], [], [], []

    def add(r, c, k, v):
        r = np.asarray(r, dtype=np.int64)
        c = np.asarray(c, dtype=np.int64)
        hi, lo = np.maximum(r, c), np.minimum(r, c)
        rows.append(hi)
        cols.append(lo)
        kind.append(np.full(hi.size, k, dtype=np.int8))
        vals.append(np.asarray(v, dtype=np.float64) * np.ones(hi.size))

    i, k = lines[:, 0], lines[:, 1]
    # H diagonal (D_x added per system)
    hdiag = np.zeros(n)
    hdiag[:2 * nbus] = rng.uniform(0.5, 2.0, 2 * nbus)
    hdiag[pg] = rng.uniform(0.1, 1.0, G)
    hdiag[qg] = rng.uniform(0.1, 1.0, G)
    add(np.arange(n), np.arange(n), 1, hdiag)
    # H couplings
    add(vm, va, 0, rng.uniform(-0.5, 0.5, nbus))
    add(va[k], va[i], 0, rng.uniform(-0.5, 0.5, L))
    add(vm[k], vm[i], 0, rng.uniform(-0.5, 0.5, L))

    def jv(size):
        return rng.choice([-1.0, 1.0], size) * rng.uniform(0.5, 2.0, size)

    # balance rows: own bus
    add(rP, va, 2, jv(nbus))
    add(rP, vm, 2, jv(nbus))
    add(rQ, vm, 2, jv(nbus))
    add(rQ, va, 2, jv(nbus))
    # neighbours (both directions of each line)
    add(rP[i], va[k], 2, jv(L))
    add(rP[k], va[i], 2, jv(L))
    add(rQ[i], vm[k], 2, jv(L))
    add(rQ[k], vm[i], 2, jv(L))
    # generators and imbalance slacks
    add(rP[gens], pg, 2, -1.0)
    add(rQ[gens], qg, 2, -1.0)
    add(rP[imb], sp, 2, 1.0)
    add(rQ[imb], sq, 2, 1.0)
    # flow-limit rows
    for rr, ss in ((rF, sf), (rT, st)):
        add(rr, va[i], 2, jv(L))
        add(rr, va[k], 2, jv(L))
        add(rr, vm[i], 2, jv(L))
        add(rr, vm[k], 2, jv(L))
        add(rr, ss, 2, 1.0)

    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    kind = np.concatenate(kind)
    raw = np.concatenate(vals)
    key = np.lexsort((cols, rows))
    rs, cs = rows[key], cols[key]
    head = np.ones(rs.size, dtype=bool)
    head[1:] = (rs[1:] != rs[:-1]) | (cs[1:] != cs[:-1])
    if not head.all():
        raise AssertionError("generator produced duplicate entries")
    pos = np.empty(rows.size, dtype=np.int64)
    pos[key] = np.arange(rows.size)
    row_ptr = np.zeros(N + 1, dtype=np.int64)
    np.cumsum(np.bincount(rs, minlength=N), out=row_ptr[1:])
    var_of_diag = np.where(kind == 1, rows, -1)
    # variable class: 0 = Va (free), 1 = Vm, 2 = Pg/Qg, 3 = flow slack, 4 = imbalance slack
    vclass = np.zeros(n, dtype=np.int8)
    vclass[vm] = 1
    vclass[pg] = 2
    vclass[qg] = 2
    vclass[sf] = 3
    vclass[st] = 3
    vclass[sp] = 4
    vclass[sq] = 4
    K = CsMatrix(N, N, row_ptr, cs, np.zeros(rs.size), SYMMETRIC_LOWER, _checked=True)
    pat = AcopfPattern(nbus=nbus, n=n, m=m, K=K, pos=pos, kind=kind,
                       var_of_diag=var_of_diag, base=raw,
                       meta=dict(nbus=nbus, lines=L, gens=G, imbalance=S, seed=seed,
                                 d_exp=ACOPF_D_EXP.get(nbus, 0.8),
                                 vclass=vclass))
    K.values = system_values(pat, 0, seed)
    return pat


# per-class probability of a bound being active at the barrier solution
ACTIVE_PROB = (0.0, 0.1, 0.3, 0.1, 0.3)
BOUNDED = (False, True, True, True, True)


MU_STEP = 0.4  # mu_k = 10**(-MU_STEP*k): calibrated so IR triggers on ~1/3 of the systems


def system_values(pat: AcopfPattern, k: int, seed: int = 0, mu_step: float = MU_STEP,
                  d_exp: float | None = None, active_prob=ACTIVE_PROB) -> np.ndarray:
    """Lower-triangle values of system ``k`` (mu_k = 10**(-mu_step*k))."""
    n = pat.n
    if k == 0:
        x = np.ones(n)
        z = np.ones(n)
        raw = pat.base.copy()
    else:
        mu = 10.0 ** (-mu_step * k)
        rng = np.random.default_rng([seed, 7919, k])
        vclass = pat.meta["vclass"]
        prob = np.asarray(active_prob)[vclass]
        active = np.random.default_rng([seed, 104729]).random(n) < prob
        if d_exp is None:  # the pattern's calibration (ACOPF_D_EXP), else 0.8
            d_exp = pat.meta.get("d_exp", 0.8)
        sm = mu ** d_exp
        x = np.where(active, sm * rng.uniform(0.5, 2.0, n), rng.uniform(0.5, 2.0, n))
        z = np.where(active, rng.uniform(0.5, 2.0, n), sm * rng.uniform(0.5, 2.0, n))
        z = np.where(np.asarray(BOUNDED)[vclass], z, 0.0)
        raw = pat.base * (1.0 + 0.01 * rng.uniform(-1.0, 1.0, pat.base.size))
    d = z / x
    isdiag = pat.kind == 1
    raw = raw.copy()
    raw[isdiag] = raw[isdiag] + d[pat.var_of_diag[isdiag]]
    vals = np.empty(pat.K.nnz)
    vals[pat.pos] = raw
    return vals


def system_rhs(pat: AcopfPattern, k: int, seed: int = 0) -> np.ndarray:
    return np.random.default_rng([seed, 31337, k]).standard_normal(pat.N)


@dataclass
class AcopfSequence:
    pattern: AcopfPattern
    seed: int
    length: int

    def mu(self, k: int) -> float:
        return 10.0 ** (-MU_STEP * k)

    def values(self, k: int) -> np.ndarray:
        return system_values(self.pattern, k, self.seed)

    def rhs(self, k: int) -> np.ndarray:
        return system_rhs(self.pattern, k, self.seed)

    def matrix(self, k: int) -> CsMatrix:
        return self.pattern.K.with_values(self.values(k))


def make_sequence(config: str | int = "activsg200", seed: int = 0, length: int = 20,
                  **kw) -> AcopfSequence:
    nbus = ACOPF_CONFIGS[config] if isinstance(config, str) else int(config)
    return AcopfSequence(build_pattern(nbus, seed, **kw), seed, length)
