"""Feasibility tests and the adaptive search, with the iteration loop on the GPU.

Public surface mirrors R/meta.py (R = /root/reference/pkg/src/symcone/):
result types (:25-205), ``iteration_bound`` (:208-213), ``early_stop_check``
(:216-235), ``solve_ftp`` (:244-395), ``refine_run`` (:457-573) and
``adaptive_search`` (:656-781).

What changed at the plugin boundary: an ``OracleSpec`` no longer carries a
Python ``query`` callback.  It carries a :class:`DeviceProblem` — the instance
resident in HBM — and ``solve_ftp`` / ``refine_run`` each become ONE call of
the C ABI ``sc_ftp`` (include/scmwu.h), which runs every iteration of the test
(learner update, oracle, width check, progress, windows, counters, early stop)
inside a single persistent CUDA kernel.  ``adaptive_search`` stays on the host
(<= 400 calls per solve, R/meta.py:449).
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field
from enum import Enum
from typing import Callable, Optional, Union

import numpy as np

from . import _native as nat
from .cones import Cone, Element


class Orientation(Enum):
    """MAX: primal max / dual min.  MIN: primal min / dual max (R/meta.py:25-30)."""
    MAX = "max"
    MIN = "min"


@dataclass(frozen=True)
class Separated:
    oracle_value: float


@dataclass(frozen=True)
class Witness:
    y: np.ndarray
    residual: Element
    candidate_value: Optional[float] = None
    oracle_value: Optional[float] = None


OracleOutcome = Union[Separated, Witness]


@dataclass(frozen=True)
class EarlyStopConfig:
    delta: float = 1e-4
    patience: int = 10
    enabled: bool = True


class DeviceIterate:
    """Lazily materialised trace-one iterate p of one sc_ftp call
    (PrimalCertificate.p / DualFeasible.p_last).  Reading ``coords`` runs one
    device pass; it is valid until the next call on the same problem."""

    def __init__(self, problem: "DeviceProblem", call_id: int):
        self.problem = problem
        self.call_id = call_id
        self.cone = problem.cone
        self._coords = None

    @property
    def coords(self) -> np.ndarray:
        if self._coords is None:
            if self.problem.handle.calls != self.call_id:
                raise RuntimeError("iterate is stale: a later feasibility test ran on this "
                                   "problem")
            self._coords = self.problem.handle.iterate()
        return self._coords

    def element(self) -> Element:
        return Element(self.cone, self.coords)


class DeviceProblem:
    """An application instance resident on the GPU plus its built-in progress
    measure (ses_progress / svm_progress).  Created by solve_ses / solve_svm."""

    def __init__(self, handle: nat.Handle, cone: Cone, kind: int):
        self.handle = handle
        self.cone = cone
        self.kind = kind
        self.best_pd_dist: Optional[float] = None   # best_pd["dist"] (R/svm.py:171)
        self.last_kernel_ms = 0.0
        self.total_kernel_ms = 0.0
        self.total_passes = 0
        self.total_width_passes = 0
        self.calls = 0

    def progress(self, y_bar) -> float:
        """Certified objective of a dual point, one device pass (R/ses.py:82-87,
        R/svm.py:87-94)."""
        return self.handle.progress(y_bar)

    def run(self, args: nat.ScFtpArgs) -> nat.FtpOut:
        out = self.handle.ftp(args)
        self.calls += 1
        self.last_kernel_ms = out.kernel_ms
        self.total_kernel_ms += out.kernel_ms
        self.total_passes += out.passes
        self.total_width_passes += out.width_passes
        if out.counter_min is not None and (self.best_pd_dist is None
                                            or out.counter_min < self.best_pd_dist):
            self.handle.pd_commit(0)
            self.best_pd_dist = out.counter_min
        return out

    def pd_pair(self):
        """(mu^, gam^, dist) of the best committed pd_counter state (SVM)."""
        return self.handle.pd_pair()

    def offer_separation(self, dist: float) -> None:
        """pd_counter(cert.p) side effect at a separation (R/svm.py:201-204)."""
        if self.best_pd_dist is None or dist < self.best_pd_dist:
            self.handle.pd_commit(1)
            self.best_pd_dist = dist

    def close(self):
        self.handle.close()


@dataclass(frozen=True)
class OracleSpec:
    """Everything a feasibility test needs (R/meta.py:63-89), with the query
    callback replaced by the device-resident problem."""

    cone: Cone
    width_rho: float
    dual_dim: int
    device: DeviceProblem
    trace_bound: float
    orientation: Orientation
    counter_progress: bool = False


@dataclass
class DualFeasible:
    y_tilde: np.ndarray
    value: float
    iterations: int
    reason: str = "exhausted"
    eps_eff: float = 0.0
    best_progress: Optional[float] = None
    best_y: Optional[np.ndarray] = None
    best_counter: Optional[float] = None
    p_last: Optional[DeviceIterate] = None
    kernel_ms: float = 0.0
    passes: int = 0


@dataclass
class PrimalCertificate:
    p: DeviceIterate
    alpha: float
    iterations: int
    oracle_value: float = 0.0
    best_progress: Optional[float] = None
    best_y: Optional[np.ndarray] = None
    best_counter: Optional[float] = None
    sep_dist: Optional[float] = None   # SVM: |P^T mu^ - Q^T gam^| of p (R/svm.py:204)
    kernel_ms: float = 0.0
    passes: int = 0


FtpResult = Union[DualFeasible, PrimalCertificate]


class Termination(Enum):
    RANGE_CONVERGED = "RangeConverged"
    EARLY_STOPPED = "EarlyStopped"
    ITERATION_CAP = "IterationCap"


@dataclass
class SearchStep:
    alpha: float
    eps: float
    iteration_bound: int
    iterations: int
    separated: bool
    reason: str


@dataclass
class SearchResult:
    lower: float
    upper: float
    best_value: float
    best_y: np.ndarray
    last_primal: Optional[PrimalCertificate]
    last_dual: Optional[DualFeasible]
    total_iterations: int
    search_steps: int
    termination: Termination
    steps: list[SearchStep] = field(default_factory=list)


@dataclass
class SolveReport:
    primal_value: float
    dual_value: float
    payload: object
    total_iterations: int
    search_steps: int
    wall_time: float
    termination: Termination
    steps: list[SearchStep] = field(default_factory=list)
    kernel_ms: float = 0.0      # sum of persistent-kernel times (CUDA events)
    passes: int = 0             # streaming passes over the point matrix
    width_passes: int = 0       # SES passes that evaluated the exact width residuals


class WidthViolationError(RuntimeError):
    def __init__(self, alpha: float, rho: float, iteration: int, norm: float):
        self.alpha, self.rho, self.iteration, self.norm = alpha, rho, iteration, norm
        super().__init__(f"residual infinity norm {norm} exceeds width {rho} "
                         f"at iteration {iteration}, level {alpha}")


def iteration_bound(trace_bound: float, width_rho: float, rank: int, eps: float,
                    alpha: float) -> int:
    """ceil(4 R^2 rho^2 ln r / (eps^2 alpha^2)), same operation order as R/meta.py:212."""
    return math.ceil(4.0 * trace_bound ** 2 * width_rho ** 2 * math.log(rank)
                     / (eps ** 2 * alpha ** 2))


def early_stop_check(history, delta: float, patience: int) -> bool:
    """R/meta.py:216-235: relative change below delta for `patience` steps."""
    if delta <= 0:
        raise ValueError("delta must be positive")
    if patience < 1:
        raise ValueError("patience must be >= 1")
    streak, prev = 0, None
    for f in history:
        if prev is not None and prev != 0.0:
            if abs(f - prev) / abs(prev) < delta:
                streak += 1
                if streak >= patience:
                    return True
            else:
                streak = 0
        prev = f
    return False


LADDER_BASE = 64
LADDER_FACTOR = 8
WINDOW_CHECK_EVERY = 16
PROGRESS_STRIDE = 4
MAX_SEARCH_STEPS = 400
BRACKET_TEST_CAP = 2048
REFINE_START = 2048
REFINE_HORIZON = 131072
MAX_REFINE_ROUNDS = 12
VALUE_TREND_DROP = 0.05

_BUDGET_CLAMP = 1 << 62


def _progress_flag(oracle: OracleSpec, progress) -> int:
    if progress is None:
        return 0
    dev = oracle.device
    if progress is dev.progress or getattr(progress, "__self__", None) is dev \
            or getattr(progress, "device_problem", None) is dev:
        return 1
    raise TypeError("progress must be None or the oracle's device progress measure: "
                    "host callbacks cannot run inside the fused device loop")


def _result(out: nat.FtpOut, oracle: OracleSpec, alpha: float) -> FtpResult:
    dev = oracle.device
    if out.status == nat.SC_EWIDTH:
        raise WidthViolationError(alpha, oracle.width_rho, out.width_iteration,
                                  out.width_norm)
    p = DeviceIterate(dev, dev.handle.calls)
    if out.kind == nat.SC_PRIMAL:
        return PrimalCertificate(p=p, alpha=alpha, iterations=out.iterations,
                                 oracle_value=out.oracle_value, best_progress=out.best_f,
                                 best_y=out.best_y, best_counter=out.best_counter,
                                 sep_dist=out.sep_dist if oracle.counter_progress else None,
                                 kernel_ms=out.kernel_ms, passes=out.passes)
    return DualFeasible(y_tilde=out.y_tilde, value=out.value, iterations=out.iterations,
                        reason=out.reason, eps_eff=out.eps_eff, best_progress=out.best_f,
                        best_y=out.best_y, best_counter=out.best_counter, p_last=p,
                        kernel_ms=out.kernel_ms, passes=out.passes)


def solve_ftp(oracle: OracleSpec, alpha: float, eps: float,
              stopping: EarlyStopConfig | None = None, progress=None,
              cap: int | None = None) -> FtpResult:
    """One feasibility test at level alpha (R/meta.py:244-395), one kernel launch."""
    if alpha <= 0:
        raise ValueError("alpha must be positive")
    if eps <= 0:
        raise ValueError("eps must be positive")
    if stopping is None:
        stopping = EarlyStopConfig()
    rank = oracle.cone.rank
    ln_r = math.log(rank)
    budget = iteration_bound(oracle.trace_bound, oracle.width_rho, rank, eps, alpha)
    if cap is not None:
        budget = min(budget, cap)
    args = nat.ScFtpArgs(mode=nat.SC_MODE_FTP, has_progress=_progress_flag(oracle, progress),
                         alpha=alpha, eps=eps, budget=max(0, min(budget, _BUDGET_CLAMP)),
                         horizon=0, ceil_ln_r=math.ceil(ln_r), delta=stopping.delta,
                         patience=stopping.patience, enabled=int(bool(stopping.enabled)),
                         gain_rel=math.nan, lo=-math.inf, hi=math.inf, target=math.nan)
    return _result(oracle.device.run(args), oracle, alpha)


def refine_run(oracle: OracleSpec, alpha: float, horizon: int, stopping: EarlyStopConfig,
               progress, gain_rel: float | None = None,
               bounds: tuple[float, float] | None = None,
               target: float | None = None) -> FtpResult:
    """Polish run at a fixed level (R/meta.py:457-573), one kernel launch."""
    if progress is None or _progress_flag(oracle, progress) != 1:
        raise TypeError("refine_run needs the oracle's device progress measure")
    rank = oracle.cone.rank
    ln_r = math.log(rank)
    horizon = max(horizon, math.ceil(ln_r))
    if gain_rel is None:
        gain_rel = stopping.delta
    lo, hi = bounds if bounds is not None else (-math.inf, math.inf)
    args = nat.ScFtpArgs(mode=nat.SC_MODE_REFINE, has_progress=1, alpha=alpha, eps=math.nan,
                         budget=0, horizon=horizon, ceil_ln_r=math.ceil(ln_r),
                         delta=stopping.delta, patience=stopping.patience,
                         enabled=int(bool(stopping.enabled)), gain_rel=gain_rel, lo=lo, hi=hi,
                         target=math.nan if target is None else target)
    return _result(oracle.device.run(args), oracle, alpha)


class _Bracket:
    """Sound bracket [L, U] plus the best certified payload (R/meta.py:576-653)."""

    def __init__(self, L: float, U: float, is_max: bool, on_primal, gain_floor: float):
        self.L, self.U, self.is_max = L, U, is_max
        self.on_primal, self.gain_floor = on_primal, gain_floor
        self.best_f: Optional[float] = None
        self.best_y: Optional[np.ndarray] = None
        self.last_primal: Optional[PrimalCertificate] = None
        self.last_dual: Optional[DualFeasible] = None

    def _tighten_from_dual_side(self, f: float) -> None:
        if self.is_max:
            self.U = min(self.U, f)
        else:
            self.L = max(self.L, f)

    def _tighten_from_primal_side(self, f: float) -> None:
        if self.is_max:
            self.L = max(self.L, f)
        else:
            self.U = min(self.U, f)

    def seed(self, f: float, y: np.ndarray) -> None:
        self.best_f, self.best_y = f, np.asarray(y)
        self._tighten_from_dual_side(f)

    def absorb(self, result: FtpResult, alpha: float) -> bool:
        span_before = self.U - self.L
        improved = False
        if isinstance(result, PrimalCertificate):
            self.last_primal = result
            self._tighten_from_primal_side(alpha)       # separation is exact
            if self.on_primal is not None:
                c = self.on_primal(result)
                if c is not None:
                    self._tighten_from_primal_side(c)
        else:
            self.last_dual = result
            self._tighten_from_dual_side(result.value)  # regret-certified claim
        if result.best_progress is not None:
            f, y = result.best_progress, result.best_y
            better = self.best_f is None or (f < self.best_f if self.is_max else f > self.best_f)
            if better:
                if self.best_f is not None and \
                        abs(self.best_f - f) > self.gain_floor * abs(self.best_f):
                    improved = True
                self.best_f, self.best_y = f, y
            self._tighten_from_dual_side(self.best_f)
        if result.best_counter is not None:
            self._tighten_from_primal_side(result.best_counter)
        return improved or (self.U - self.L) < span_before * (1.0 - 2e-2)

    def span(self) -> float:
        return self.U - self.L

    def converged(self, eps: float) -> bool:
        span = self.span()
        if self.L > 0.0:
            ref = self.L
        else:
            ref = span / 3.0 if self.is_max else 2.0 * span / 3.0
        return span < eps * ref


def host_search_requested() -> bool:
    """SCMWU_HOST_SEARCH=1: drive the adaptive search from the host, one launch per test
    (the round-1 path; kept for A/B and for the parity tests of the device search)."""
    return os.environ.get("SCMWU_HOST_SEARCH", "0") not in ("", "0")


def resident_search(oracle: OracleSpec, L0: float, U0: float, eps: float,
                    stopping: EarlyStopConfig | None, cap: int | None,
                    seed_y: np.ndarray, on_primal: bool = False,
                    zero_lower_floor: float | None = None,
                    refine_horizon: int = REFINE_HORIZON):
    """adaptive_search (R/meta.py:656-781) with the bracket, every test and the seed /
    final progress passes inside ONE persistent kernel launch (sc_solve).  The seed
    certificate is (progress(seed_y), (seed_y; f)) for SES and (progress(w0), (w0; 0; 0))
    for SVM, exactly as solve_ses / solve_svm build it.  Returns (SearchResult, seed_f,
    final_f): final_f is the progress at the returned centre (SES, R/ses.py:187)."""
    if not 0.0 <= L0 < U0:
        raise ValueError(f"need 0 <= L0 < U0, got [{L0}, {U0}]")
    if not 0.0 < eps < 1.0:
        raise ValueError("eps must be in (0, 1)")
    if stopping is None:
        stopping = EarlyStopConfig()
    dev = oracle.device
    ln_r = math.log(oracle.cone.rank)
    args = nat.ScSolveArgs(eps=eps, L0=float(L0), U0=float(U0), delta=stopping.delta,
                           patience=stopping.patience, enabled=int(bool(stopping.enabled)),
                           cap=-1 if cap is None else int(cap), ceil_ln_r=math.ceil(ln_r),
                           refine_horizon=refine_horizon,
                           zero_lower_floor=(math.nan if zero_lower_floor is None
                                             else zero_lower_floor),
                           on_primal=int(bool(on_primal)), max_steps=nat.MAX_SEARCH_STEPS)
    st, r, best_y, steps = dev.handle.solve(args, seed_y)
    dev.calls += 1
    dev.last_kernel_ms = float(r.kernel_ms)
    dev.total_kernel_ms += float(r.kernel_ms)
    dev.total_passes += int(r.passes)
    dev.total_width_passes += int(r.width_passes)
    if st == nat.SC_EWIDTH:
        raise WidthViolationError(r.width_alpha, oracle.width_rho, int(r.width_iteration),
                                  r.width_norm)
    if r.has_pd:
        dev.best_pd_dist = float(r.pd_dist)
    if not r.has_best:
        raise RuntimeError("search finished without any certified solution; "
                           "pass an initial_certificate")
    log = [SearchStep(s.alpha, s.eps, int(s.iteration_bound), int(s.iterations),
                      bool(s.separated), nat.REASONS.get(s.reason, "?")) for s in steps]
    res = SearchResult(lower=r.lower, upper=r.upper, best_value=r.best_value, best_y=best_y,
                       last_primal=None, last_dual=None,
                       total_iterations=int(r.total_iterations),
                       search_steps=int(r.search_steps),
                       termination=Termination(nat.SC_TERMINATIONS[r.termination]), steps=log)
    return res, float(r.seed_f), float(r.final_f)


def adaptive_search(oracle_factory: Callable[[float], OracleSpec], L0: float, U0: float,
                    eps: float, stopping: EarlyStopConfig | None = None, progress=None,
                    cap: int | None = None,
                    initial_certificate: tuple[float, np.ndarray] | None = None,
                    on_primal: Callable[[PrimalCertificate], float | None] | None = None,
                    zero_lower_floor: float | None = None,
                    refine_horizon: int = REFINE_HORIZON) -> SearchResult:
    """Bracket, then polish (R/meta.py:656-781).  Host-side driver; every test
    it issues is one device call."""
    if not 0.0 <= L0 < U0:
        raise ValueError(f"need 0 <= L0 < U0, got [{L0}, {U0}]")
    if not 0.0 < eps < 1.0:
        raise ValueError("eps must be in (0, 1)")
    if stopping is None:
        stopping = EarlyStopConfig()
    is_max = oracle_factory((L0 + U0) / 2.0).orientation is Orientation.MAX
    br = _Bracket(float(L0), float(U0), is_max, on_primal, max(stopping.delta, eps / 10.0))
    if initial_certificate is not None:
        br.seed(*initial_certificate)
    total = 0
    steps: list[SearchStep] = []
    capped = floored = False
    test_cap = min(BRACKET_TEST_CAP, cap) if cap is not None else BRACKET_TEST_CAP

    # bracketing phase (R/meta.py:705-730)
    while len(steps) < MAX_SEARCH_STEPS:
        if br.converged(eps):
            break
        span = br.span()
        if zero_lower_floor is not None and br.L == 0.0 and span < zero_lower_floor:
            floored = True
            break
        alpha = br.L + span / 3.0 if is_max else br.L + 2.0 * span / 3.0
        eps_i = span / (3.0 * alpha)
        oracle = oracle_factory(alpha)
        T_i = iteration_bound(oracle.trace_bound, oracle.width_rho, oracle.cone.rank, eps_i,
                              alpha)
        res = solve_ftp(oracle, alpha, eps_i, stopping, progress, test_cap)
        total += res.iterations
        if cap is not None and cap < T_i and isinstance(res, DualFeasible) \
                and res.reason == "exhausted" and res.iterations >= cap:
            capped = True
        productive = br.absorb(res, alpha)
        steps.append(SearchStep(alpha, eps_i, T_i, res.iterations,
                                isinstance(res, PrimalCertificate),
                                getattr(res, "reason", "separated")))
        if not productive:
            break

    # polish phase (R/meta.py:732-763)
    if progress is not None and not floored:
        h = REFINE_START
        for _ in range(MAX_REFINE_ROUNDS):
            if br.converged(eps) or len(steps) >= MAX_SEARCH_STEPS:
                break
            alpha = (br.L + br.U) / 2.0
            if alpha <= 0.0:
                break
            oracle = oracle_factory(alpha)
            T_i = iteration_bound(oracle.trace_bound, oracle.width_rho, oracle.cone.rank, eps,
                                  alpha)
            full = min(T_i, refine_horizon) if cap is None else min(T_i, refine_horizon, cap)
            horizon = min(h, full)
            res = refine_run(oracle, alpha, horizon, stopping, progress,
                             gain_rel=max(stopping.delta, eps / 20.0), bounds=(br.L, br.U),
                             target=eps)
            total += res.iterations
            productive = br.absorb(res, alpha)
            steps.append(SearchStep(alpha, eps, T_i, res.iterations,
                                    isinstance(res, PrimalCertificate),
                                    getattr(res, "reason", "separated")))
            if not productive and horizon >= full:
                break
            h = min(h * 4, refine_horizon)

    if br.best_f is None or br.best_y is None:
        raise RuntimeError("search finished without any certified solution; "
                           "pass an initial_certificate")
    if capped:
        term = Termination.ITERATION_CAP
    elif br.converged(eps):
        term = Termination.RANGE_CONVERGED
    else:
        term = Termination.EARLY_STOPPED
    return SearchResult(lower=br.L, upper=br.U, best_value=br.best_f, best_y=br.best_y,
                        last_primal=br.last_primal, last_dual=br.last_dual,
                        total_iterations=total, search_steps=len(steps), termination=term,
                        steps=steps)
