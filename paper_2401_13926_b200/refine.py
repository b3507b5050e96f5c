"""Drop-in for ``kktsolve.refine``: FGMRES and Richardson iterative refinement on the B200.

``refine_fgmres`` follows refine.py:103-132 step for step — trigger, NSR before, FGMRES
with the (stale) LU factors as right preconditioner and ``tol = delta_tol``, NSR/NRBE after —
with every vector operation on the device.  The quality metrics come from one fused device
pass (``kkt_dev_residual_norms``) instead of separate host spmv calls.

Barrier-tied tolerance (the north star's extension; the reference fixes ``delta_tol``,
SURVEY.md §5): :class:`BarrierTiedTolerance` maps the interior-point parameter mu to
``delta(mu) = clamp(theta * mu, delta_min, delta_max)``; :class:`FixedTolerance` is the
reference behaviour and the parity default.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

from .krylov import KrylovConfig

NSR_RATIO = "nsr_ratio"
TOLERANCE = "tolerance"


@dataclass
class RefinementConfig:
    """Trigger tolerance + per-method knobs (refine.py:26-45)."""

    delta_tol: float = 1e-9
    krylov: KrylovConfig = field(default_factory=KrylovConfig)
    richardson_max_steps: int = 10
    richardson_stop: str = TOLERANCE
    nsr_ratio_floor: float = 0.5

    def __post_init__(self):
        if self.delta_tol <= 0:
            raise ValueError("delta_tol must be positive")
        if self.richardson_stop not in (TOLERANCE, NSR_RATIO):
            raise ValueError(f"unknown richardson_stop {self.richardson_stop!r}")


@dataclass
class RefinementReport:
    triggered: bool
    method: str
    ir_iterations: int
    triangular_solves_used: int
    nsr_before: float
    nsr_after: float
    rr_final: float
    nrbe_final: float
    converged: bool
    diverged: bool = False


@dataclass(frozen=True)
class FixedTolerance:
    """The reference policy: one delta for every system."""

    delta: float = 1e-9

    def __call__(self, mu: float | None = None) -> float:
        return self.delta


@dataclass(frozen=True)
class BarrierTiedTolerance:
    """delta(mu) = clamp(theta * mu, delta_min, delta_max).

    Defaults 1e-2 / 1e-10 / 1e-8: the paper's IR tolerances span 1e-9..1e-10;
    at N~238k the FGMRES floor sits near 1e-12..1e-14 relative, so tighter minima exhaust
    the restart budget on the last barrier systems (measured with the oracle).

    Loose while the barrier parameter is large (early, well-conditioned systems need no
    refinement), tight as mu -> 0 where the static-pivot factors degrade.
    """

    theta: float = 1e-2
    delta_min: float = 1e-10
    delta_max: float = 1e-8

    def __post_init__(self):
        if not (self.theta > 0 and 0 < self.delta_min <= self.delta_max):
            raise ValueError("need theta > 0 and 0 < delta_min <= delta_max")

    def __call__(self, mu: float | None = None) -> float:
        if mu is None:
            return self.delta_max
        return float(min(max(self.theta * float(mu), self.delta_min), self.delta_max))


def config_for_mu(cfg: RefinementConfig, policy, mu: float | None) -> RefinementConfig:
    """The refinement config for one system of a barrier sequence."""
    return replace(cfg, delta_tol=policy(mu))


def _stats(K, x, r):
    from .sparse_ops import residual_stats
    return residual_stats(K, r, x)


def nsr(K, x, r) -> float:
    """||r - Kx||_inf / (||K||_inf ||x||_inf), +inf for a zero denominator (refine.py:62)."""
    return _stats(K, x, r).nsr()


def nrbe(K, x, r) -> float:
    """||r - Kx||_2 / (||K||_inf ||x||_2 + ||r||_2) (refine.py:76)."""
    return _stats(K, x, r).nrbe()


def needs_refinement(K, x0, r, delta_tol: float) -> bool:
    """||r - K x0||_2 > delta_tol * ||r||_2 (refine.py:88)."""
    s = _stats(K, x0, r)
    return s.err2 > delta_tol * s.r2


def refine_fgmres(K, factors, x0, r, cfg: RefinementConfig):
    """FGMRES refinement of a direct solve, LU factors as right preconditioner (refine.py:103).

    One device call (``kkt_dev_refine_fgmres``): the trigger ``||r - K x0||_2 > delta ||r||_2``
    (:113), NSR before (:117), FGMRES with ``tol = delta_tol`` (:119-126) and NSR / NRBE after
    (:129-131) are all computed and decided on the device; the host synchronises once.
    """
    from .device import ResidualStats
    x0 = np.asarray(x0, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    dev = factors.device(restart_m=cfg.krylov.m)
    dev.set_operator(K)
    dev.h2d(dev.r, r)
    dev.h2d(dev.x0, x0)
    if cfg.krylov.ortho not in ("cgs2", "mgs"):
        raise ValueError(f"unknown orthogonalization {cfg.krylov.ortho!r}")
    rep = dev.refine_device(dev.r, dev.x0, dev.x, cfg.krylov.m, cfg.krylov.max_outer, cfg.delta_tol,
                            mgs=cfg.krylov.ortho == "mgs")
    s0 = ResidualStats(*rep.stats_before)
    if not rep.triggered:                                                    # (:113-114)
        q = s0.nsr()
        return x0.copy(), RefinementReport(
            triggered=False, method="none", ir_iterations=0, triangular_solves_used=0,
            nsr_before=q, nsr_after=q, rr_final=1.0, nrbe_final=s0.nrbe(), converged=True)
    count0 = factors.triangular_solve_count
    factors.triangular_solve_count += rep.precond_applications
    s1 = ResidualStats(*rep.stats_after)
    x = dev.d2h(dev.x)
    rho0 = rep.beta0
    rr_final = (rep.est_final / rho0) if rho0 > 0 else 0.0               # (:123-124)
    return x, RefinementReport(
        triggered=True, method="fgmres", ir_iterations=rep.iterations,
        triangular_solves_used=factors.triangular_solve_count - count0,
        nsr_before=s0.nsr(), nsr_after=s1.nsr(), rr_final=rr_final, nrbe_final=s1.nrbe(),
        converged=bool(rep.converged))


def refine_richardson(K, factors, x0, r, cfg: RefinementConfig):
    """Richardson iterative refinement (refine.py:135-205) with every vector on the device.

    Per step: d = lu_solve(rho) (device trisolves), x += d (device), rho = r - K x with its
    2-norm (one fused device pass).  The stopping rules are the reference's: residual
    tolerance or NSR stagnation, the step budget, divergence after two consecutive residual
    increases (then the best iterate is returned).  The host reads one norm per step.
    """
    x0 = np.asarray(x0, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    dev = factors.device(restart_m=cfg.krylov.m)
    torch = dev.torch
    dev.set_operator(K)
    dev.h2d(dev.r, r)
    dev.h2d(dev.x0, x0)
    s0 = dev.residual_stats_device(dev.r, dev.x0)
    if not (s0.err2 > cfg.delta_tol * s0.r2):                      # :147-148
        q = s0.nsr()
        return x0.copy(), RefinementReport(
            triggered=False, method="none", ir_iterations=0, triangular_solves_used=0,
            nsr_before=q, nsr_after=q, rr_final=1.0, nrbe_final=s0.nrbe(), converged=True)
    count0 = factors.triangular_solve_count
    nsr_before = s0.nsr()
    r_norm = s0.r2
    with torch.cuda.stream(dev.stream):
        x = dev.x0.clone()
        rho = torch.empty_like(x)
        dvec = torch.empty_like(x)
        best_x = x.clone()
    rho_norm = dev.residual_device(dev.r, x, rho)                  # :158
    rho0_norm = rho_norm
    nsr_old = nsr_before
    best_rho = rho_norm
    steps, converged, diverged, growth = 0, False, False, 0
    while steps < cfg.richardson_max_steps:
        if cfg.richardson_stop == TOLERANCE and rho_norm <= cfg.delta_tol * r_norm:
            converged = True
            break
        dev.solve_device(rho, dvec)                                # :166  d = lu_solve(rho)
        factors.triangular_solve_count += 1
        dev.axpy_device(x, dvec)                                   #       x += d
        steps += 1
        new_norm = dev.residual_device(dev.r, x, rho)              # :168
        if new_norm < best_rho:
            with torch.cuda.stream(dev.stream):
                best_x.copy_(x)
            best_rho = new_norm
        if new_norm > rho_norm:
            growth += 1
            if growth >= 2:
                diverged = True
                break
        else:
            growth = 0
        rho_norm = new_norm
        if cfg.richardson_stop == NSR_RATIO:
            nsr_new = dev.residual_stats_device(dev.r, x).nsr()
            if nsr_old > 0 and nsr_new / nsr_old > cfg.nsr_ratio_floor:
                converged = True
                break
            nsr_old = nsr_new
    else:
        converged = cfg.richardson_stop == TOLERANCE and rho_norm <= cfg.delta_tol * r_norm
    if diverged:
        x, rho_norm = best_x, best_rho
    s1 = dev.residual_stats_device(dev.r, x)
    xh = dev.d2h(x)
    return xh, RefinementReport(
        triggered=True, method="richardson", ir_iterations=steps,
        triangular_solves_used=factors.triangular_solve_count - count0,
        nsr_before=nsr_before, nsr_after=s1.nsr(),
        rr_final=(rho_norm / rho0_norm) if rho0_norm > 0 else 0.0,
        nrbe_final=s1.nrbe(), converged=converged, diverged=diverged)
