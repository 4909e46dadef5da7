"""numpy + C restatement of the reference SCMWU path — TEST INFRASTRUCTURE ONLY.

Every function cites the reference lines it restates (R = /root/reference/
pkg/src/symcone/).  Arithmetic is kept in the reference's order so that, on
the same machine, the oracle reproduces the reference bit for bit at
threads=1 (pinned by tests/test_oracle_golden.py against fixtures produced by
tests/golden/make_golden.py):

  * SOC loops (eigenvalue bound, exp run, infinity norm) run in C with glibc
    exp and sequential sums (soc_kernels.c), as the reference's numba loops do;
  * numpy reductions / BLAS products are issued with the same numpy calls on
    the same array shapes as the reference.

The oracle stores the O(n d) cumulative loss like the reference does; the
CUDA path does not (it uses the closed form).  It is the checker
and the CPU baseline, never a fallback for the product.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

SQRT2 = math.sqrt(2.0)

# control constants, verbatim from the reference
LOSS_SLACK = 1e-9                 # R/mwu.py:23
LADDER_BASE, LADDER_FACTOR = 64, 8  # R/meta.py:238-239
CHECK_EVERY, PROGRESS_STRIDE = 16, 4  # R/meta.py:240-241
MAX_SEARCH_STEPS = 400            # R/meta.py:449
BRACKET_TEST_CAP = 2048           # R/meta.py:450
REFINE_START, REFINE_HORIZON = 2048, 131072  # R/meta.py:451-452
MAX_REFINE_ROUNDS = 12            # R/meta.py:453
VALUE_TREND_DROP = 0.05           # R/meta.py:454
SVM_INFEASIBLE_FLOOR = 1e-9       # R/svm.py:145
SVM_SEARCH_EPS_FACTOR = 0.4       # R/svm.py:150

# ------------------------------------------------------------------ C kernels
_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle_soc.so")
_lib = None


def build_oracle_lib() -> str:
    """Compile soc_kernels.c (gcc, -ffp-contract=off) into oracle/_build/."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _soc():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build_oracle_lib()
        lib = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        i64 = ctypes.c_int64
        lib.orc_soc_lambda_max.argtypes = [dp, i64, i64]
        lib.orc_soc_lambda_max.restype = ctypes.c_double
        lib.orc_soc_inf_norm.argtypes = [dp, i64, i64]
        lib.orc_soc_inf_norm.restype = ctypes.c_double
        lib.orc_soc_exp_run.argtypes = [dp, dp, i64, i64, ctypes.c_double]
        lib.orc_soc_exp_run.restype = ctypes.c_double
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


# ------------------------------------------------------------------ cone iterates
def soc_normalized_exp(x: np.ndarray, w: int) -> np.ndarray:
    """normalized_exp on a cone made of one run of equal SOC blocks
    (R/cones.py:399-420 with _lambda_max :388-396 and _soc_exp_run :252-274)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    k = x.shape[0] // w
    lib = _soc()
    shift = lib.orc_soc_lambda_max(_ptr(x), k, w)
    out = np.empty_like(x)
    tr = 0.0
    tr += lib.orc_soc_exp_run(_ptr(x), _ptr(out), k, w, shift)
    if not tr > 0.0:
        raise ValueError(f"trace must be positive to normalize, got {tr}")
    out /= tr
    return out


def orthant_normalized_exp(x: np.ndarray) -> np.ndarray:
    """normalized_exp on a single orthant run (R/cones.py:399-420, :410-412)."""
    shift = float(x.max())
    out = np.empty_like(x)
    tr = 0.0
    np.exp(x - shift, out=out)
    tr += float(out.sum())
    if not tr > 0.0:
        raise ValueError(f"trace must be positive to normalize, got {tr}")
    out /= tr
    return out


def soc_inf_norm(x: np.ndarray, w: int) -> float:
    """inf_norm on one SOC run (R/cones.py:349-361, :237-249)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    return max(0.0, _soc().orc_soc_inf_norm(_ptr(x), x.shape[0] // w, w))


def orthant_inf_norm(x: np.ndarray) -> float:
    return max(0.0, float(np.abs(x).max()))


class LossNormError(ValueError):
    def __init__(self, norm: float):
        self.norm = norm
        super().__init__(f"loss infinity norm {norm} exceeds 1 + {LOSS_SLACK}")


class Learner:
    """Scmwu restated (R/mwu.py:38-70): stores the cumulative loss."""

    def __init__(self, ambient: int, eta: float, soc_width: Optional[int]):
        if not 0.0 < eta <= 1.0:
            raise ValueError(f"eta must be in (0, 1], got {eta}")
        self.eta = float(eta)
        self.w = soc_width            # None => orthant
        self.cum = np.zeros(ambient)

    def observe(self, loss: np.ndarray, prescale: float) -> None:
        nrm = (orthant_inf_norm(loss) if self.w is None
               else soc_inf_norm(loss, self.w)) * abs(prescale)
        if nrm > 1.0 + LOSS_SLACK:
            raise LossNormError(nrm)
        self.cum += prescale * loss        # R/mwu.py:15-18 (mul then add)

    def current(self) -> np.ndarray:
        x = -self.eta * self.cum
        return (orthant_normalized_exp(x) if self.w is None
                else soc_normalized_exp(x, self.w))


def part_sum(a, parts=1, axis=0):
    """R/_reduce.py:12-17."""
    if parts <= 1:
        return a.sum(axis=axis)
    return np.add.reduce(np.stack([c.sum(axis=axis)
                                   for c in np.array_split(a, parts, axis=axis)]), axis=0)


def part_matvec(m, v, parts=1):
    """R/_reduce.py:20-26."""
    if parts <= 1:
        return m.T @ v
    idx = np.array_split(np.arange(m.shape[0]), parts)
    return np.add.reduce(np.stack([m[i].T @ v[i] for i in idx]), axis=0)


# ------------------------------------------------------------------ oracle outcomes
@dataclass
class Sep:
    value: float


@dataclass
class Wit:
    y: np.ndarray
    residual: np.ndarray
    candidate: Optional[float]
    value: Optional[float]


@dataclass
class Spec:
    """What a feasibility test needs (R/meta.py:63-89)."""
    ambient: int
    soc_width: Optional[int]
    rank: int
    rho: float
    R: float
    is_max: bool
    dual_dim: int
    query: Callable
    counter: Optional[Callable] = None


# ------------------------------------------------------------------ SES
class SesProblem:
    """R/ses.py: range :65-72, progress :82-87, oracle :90-132."""

    def __init__(self, centers, radii, parts: int = 1):
        self.c = np.asarray(centers, dtype=np.float64)
        self.r = np.asarray(radii, dtype=np.float64)
        self.n, self.d = self.c.shape
        self.parts = parts
        self.buf = np.empty((self.n - 1) * (self.d + 1))

    def range(self):
        D = float((np.linalg.norm(self.c[1:] - self.c[0], axis=1)
                   + self.r[0] + self.r[1:]).max())
        return D, D / 2.0, D

    def progress(self, u):
        diff = self.c - u
        return float((np.sqrt(np.einsum("ij,ij->i", diff, diff)) + self.r).max())

    def query(self, p: np.ndarray, alpha: float):
        v1, g1 = self.c[0], float(self.r[0])
        if alpha < g1:
            return Sep(-math.inf)
        d, k = self.d, self.n - 1
        blocks = p.reshape(k, d + 1)
        Wv, sig = blocks[:, :d], blocks[:, d]
        s = np.asarray(part_sum(Wv, self.parts, 0))
        sn = float(np.linalg.norm(s))
        u = v1 + (alpha - g1) * (s / sn) if sn > 0.0 else v1.copy()
        V, g = self.c[1:], self.r[1:]
        lin = float(part_sum(np.einsum("ij,ij->i", V, Wv), self.parts))
        rad = float(part_sum(g * sig, self.parts))
        value = float(s @ u) + alpha / SQRT2 - lin - rad
        if value < 0.0:
            return Sep(value)
        res = self.buf.reshape(k, d + 1)
        np.subtract(u, V, out=res[:, :d])
        np.subtract(alpha, g, out=res[:, d])
        return Wit(np.concatenate([u, [alpha]]), self.buf, None, value)

    def spec(self, rho: float) -> Spec:
        k = self.n - 1
        return Spec(k * (self.d + 1), self.d + 1, 2 * k, rho, SQRT2, True, self.d + 1,
                    self.query)


# ------------------------------------------------------------------ SVM
class SvmProblem:
    """R/svm.py: max_norm :62-66, progress :87-94, oracle :97-127,
    extract_pd :130-137, pd_counter :173-181."""

    def __init__(self, P, Q, parts: int = 1):
        self.P = np.asarray(P, dtype=np.float64)
        self.Q = np.asarray(Q, dtype=np.float64)
        self.n1, self.d = self.P.shape
        self.n2 = self.Q.shape[0]
        self.parts = parts
        self.D = float(max(np.linalg.norm(self.P, axis=1).max(),
                           np.linalg.norm(self.Q, axis=1).max()))
        self.best_dist = None
        self.best_pair = None

    def progress(self, w):
        nrm = float(np.linalg.norm(w))
        if nrm == 0.0:
            return 0.0
        return max(float((self.P @ w).min() - (self.Q @ w).max()) / nrm, 0.0)

    def query(self, p: np.ndarray, alpha: float):
        n1, d, D = self.n1, self.d, self.D
        mu, gam = p[:n1], p[n1:]
        g = np.asarray(part_matvec(self.P, mu, self.parts)
                       - part_matvec(self.Q, gam, self.parts))
        gn = float(np.linalg.norm(g))
        if gn > 0.0:
            w = g / gn
        else:
            w = np.zeros(d)
            w[0] = 1.0
        tm, tg = float(mu.sum()), float(gam.sum())
        s1 = D if tm <= tg else alpha - D
        s2 = alpha - s1
        value = float(g @ w) - tm * s1 - tg * s2
        if value < 0.0:
            return Sep(value)
        res = np.concatenate([self.P @ w - s1, -(self.Q @ w) - s2])
        cand = float(res[:n1].min() + res[n1:].min()) + alpha
        return Wit(np.concatenate([w, [s1, s2]]), res, max(cand, 0.0), value)

    def extract_pd(self, p):
        mu, gam = p[:self.n1], p[self.n1:]
        smu, sg = float(mu.sum()), float(gam.sum())
        if smu <= 0.0 or sg <= 0.0:
            raise ValueError("both parts must have positive sums")
        return mu / smu, gam / sg

    def counter(self, p):
        mu, gam = self.extract_pd(p)
        z = self.P.T @ mu - self.Q.T @ gam
        dist = float(np.linalg.norm(z))
        if self.best_dist is None or dist < self.best_dist:
            self.best_dist, self.best_pair = dist, (mu, gam)
        return dist, np.concatenate([z, [0.0, 0.0]])

    def spec(self) -> Spec:
        n = self.n1 + self.n2
        return Spec(n, None, n, 2.0 * self.D, 2.0, False, self.d + 2, self.query,
                    self.counter)


# ------------------------------------------------------------------ results
@dataclass
class Primal:
    p: np.ndarray
    alpha: float
    iterations: int
    oracle_value: float = 0.0
    best_progress: Optional[float] = None
    best_y: Optional[np.ndarray] = None
    best_counter: Optional[float] = None


@dataclass
class Dual:
    y_tilde: np.ndarray
    value: float
    iterations: int
    reason: str = "exhausted"
    eps_eff: float = 0.0
    best_progress: Optional[float] = None
    best_y: Optional[np.ndarray] = None
    best_counter: Optional[float] = None
    p_last: Optional[np.ndarray] = None


class WidthViolation(RuntimeError):
    def __init__(self, alpha, rho, iteration, norm):
        self.alpha, self.rho, self.iteration, self.norm = alpha, rho, iteration, norm
        super().__init__(f"residual infinity norm {norm} exceeds width {rho} "
                         f"at iteration {iteration}, level {alpha}")


def iteration_bound(R, rho, rank, eps, alpha) -> int:
    """R/meta.py:208-213 (same operation order)."""
    return math.ceil(4.0 * R ** 2 * rho ** 2 * math.log(rank) / (eps ** 2 * alpha ** 2))


class Best:
    """_ProgressState (R/meta.py:398-429)."""

    def __init__(self, is_max):
        self.is_max = is_max
        self.f = None
        self.y = None
        self.counter = None

    def offer(self, f, y):
        if self.f is None or (f < self.f if self.is_max else f > self.f):
            self.f, self.y = f, y.copy()

    def offer_counter(self, v):
        if self.counter is None or (v > self.counter if self.is_max else v < self.counter):
            self.counter = v

    def beats(self, alpha):
        return self.f is not None and (self.f < alpha if self.is_max else self.f > alpha)


def _claim(eps_eff, alpha, is_max):
    """R/meta.py:432-433."""
    return (1.0 + eps_eff) * alpha if is_max else (1.0 - eps_eff) * alpha


def _dual(spec, y_bar, value, iters, reason, eps_eff, alpha, best, p):
    """R/meta.py:436-446."""
    if y_bar is None:
        y_bar = np.zeros(spec.dual_dim)
        eps_eff = math.inf
    yt = np.asarray(y_bar, dtype=np.float64).copy()
    sh = min(eps_eff, 1.0) * alpha / spec.R
    yt[-1] += sh if spec.is_max else -sh
    return Dual(yt, value, iters, reason, eps_eff, best.f, best.y, best.counter, p)


class _Window:
    """Suffix window of witnesses (R/meta.py:304-306, :330-335)."""

    def __init__(self, dim):
        self.items = []
        self.head = 0
        self.sum = np.zeros(dim)

    def push(self, y, t):
        self.items.append(y)
        self.sum += y
        while len(self.items) - self.head > max(LADDER_BASE, t // 2):
            self.sum -= self.items[self.head]
            self.items[self.head] = None
            self.head += 1

    def mean(self):
        return self.sum / (len(self.items) - self.head)


def ftp(spec: Spec, alpha, eps, delta=1e-4, patience=10, enabled=True,
        progress=None, cap=None):
    """solve_ftp restated (R/meta.py:244-395)."""
    if alpha <= 0:
        raise ValueError("alpha must be positive")
    if eps <= 0:
        raise ValueError("eps must be positive")
    ln_r = math.log(spec.rank)
    R, rho, is_max = spec.R, spec.rho, spec.is_max
    inv_rho = 1.0 / rho
    budget = iteration_bound(R, rho, spec.rank, eps, alpha)
    if cap is not None:
        budget = min(budget, cap)
    spent = 0
    rung_T = min(budget, max(LADDER_BASE, math.ceil(ln_r)))
    best = Best(is_max)
    claim_eps, claim_y = math.inf, None
    p = None
    rung = 0
    while spent < budget:
        remaining = budget - spent
        if remaining < ln_r:
            break
        rung_T = min(rung_T, remaining)
        eta = math.sqrt(ln_r / rung_T)
        learner = Learner(spec.ambient, eta, spec.soc_width)
        y_sum = np.zeros(spec.dual_dim)
        win = _Window(spec.dual_dim)
        f_prev, streak, early = None, 0, False
        f_start = best.f
        t = 0
        for t in range(1, rung_T + 1):
            p = learner.current()
            out = spec.query(p, alpha)
            if isinstance(out, Sep):
                return Primal(p, alpha, spent + t, out.value, best.f, best.y, best.counter)
            y_sum += out.y
            try:
                learner.observe(out.residual, inv_rho)
            except LossNormError as exc:
                raise WidthViolation(alpha, rho, spent + t, exc.norm * rho) from exc
            if progress is None:
                continue
            win.push(out.y, t)
            if out.candidate is not None:
                best.offer(out.candidate, out.y)
            y_bar = y_sum / t
            f = progress(y_bar)
            best.offer(f, y_bar)
            if t % CHECK_EVERY == 0 or t == rung_T or t == 1:
                yw = win.mean()
                best.offer(progress(yw), yw)
                if spec.counter is not None:
                    cv, yc = spec.counter(p)
                    best.offer_counter(cv)
                    if yc is not None:
                        best.offer(progress(yc), yc)
            if best.beats(alpha):
                return _dual(spec, best.y, best.f, spent + t, "affirmative", 0.0, alpha,
                             best, p)
            if enabled:
                if f_prev is not None and f_prev != 0.0:
                    if abs(f - f_prev) / abs(f_prev) < delta:
                        streak += 1
                        if streak >= patience:
                            early = True
                            break
                    else:
                        streak = 0
                f_prev = f
        spent += t
        e_here = R * rho * (eta + ln_r / (eta * t)) / alpha
        if e_here < claim_eps:
            claim_eps, claim_y = e_here, y_sum / t
        if claim_eps <= eps:
            return _dual(spec, claim_y, _claim(claim_eps, alpha, is_max), spent,
                         "exhausted", claim_eps, alpha, best, p)
        if early and rung >= 1 and progress is not None:
            if (f_start is not None and best.f is not None
                    and abs(f_start - best.f) <= delta * abs(f_start)):
                return _dual(spec, claim_y, _claim(claim_eps, alpha, is_max), spent,
                             "early_stop", claim_eps, alpha, best, p)
        rung += 1
        rung_T = min(remaining, rung_T * LADDER_FACTOR)
    return _dual(spec, claim_y, _claim(claim_eps, alpha, is_max), max(spent, 1),
                 "exhausted", claim_eps, alpha, best, p)


def refine(spec: Spec, alpha, horizon, delta, patience, enabled, progress,
           gain_rel=None, bounds=None, target=None):
    """refine_run restated (R/meta.py:457-573)."""
    ln_r = math.log(spec.rank)
    R, rho, is_max = spec.R, spec.rho, spec.is_max
    horizon = max(horizon, math.ceil(ln_r))
    eta = math.sqrt(ln_r / horizon)
    stall_floor = max(64 * patience, math.ceil(16.0 / eta))
    if gain_rel is None:
        gain_rel = delta
    learner = Learner(spec.ambient, eta, spec.soc_width)
    y_sum = np.zeros(spec.dual_dim)
    win = _Window(spec.dual_dim)
    best = Best(is_max)
    anchor = val_anchor = None
    last_gain = 0
    lo, hi = bounds if bounds is not None else (-math.inf, math.inf)
    p = None
    t = 0
    for t in range(1, horizon + 1):
        p = learner.current()
        out = spec.query(p, alpha)
        if isinstance(out, Sep):
            return Primal(p, alpha, t, out.value, best.f, best.y, best.counter)
        y_sum += out.y
        try:
            learner.observe(out.residual, 1.0 / rho)
        except LossNormError as exc:
            raise WidthViolation(alpha, rho, t, exc.norm * rho) from exc
        win.push(out.y, t)
        if out.candidate is not None:
            best.offer(out.candidate, out.y)
        if t % PROGRESS_STRIDE == 0 or t == 1 or t == horizon:
            y_bar = y_sum / t
            best.offer(progress(y_bar), y_bar)
        if t % CHECK_EVERY == 0 or t == horizon or t == 1:
            yw = win.mean()
            best.offer(progress(yw), yw)
            if spec.counter is not None:
                cv, yc = spec.counter(p)
                best.offer_counter(cv)
                if yc is not None:
                    best.offer(progress(yc), yc)
        gained = False
        if anchor is None or (best.f is not None
                              and abs(best.f - anchor) > gain_rel * abs(anchor)):
            anchor = best.f
            gained = True
        if out.value is not None:
            v = out.value
            if val_anchor is None:
                val_anchor = v
            elif v < val_anchor - VALUE_TREND_DROP * abs(val_anchor):
                val_anchor = v
                gained = True
        if gained:
            last_gain = t
        elif enabled and t - last_gain > max(stall_floor, t // 3):
            break
        if target is not None and t % PROGRESS_STRIDE == 0:
            if best.f is not None:
                if is_max:
                    hi = min(hi, best.f)
                else:
                    lo = max(lo, best.f)
            if best.counter is not None:
                if is_max:
                    lo = max(lo, best.counter)
                else:
                    hi = min(hi, best.counter)
            if hi - lo <= target * max(lo, 0.0):
                break
    eps_eff = R * rho * (eta + ln_r / (eta * t)) / alpha
    return _dual(spec, y_sum / t, _claim(eps_eff, alpha, is_max), t, "refined", eps_eff,
                 alpha, best, p)


# ------------------------------------------------------------------ adaptive search
@dataclass
class StepRec:
    alpha: float
    eps: float
    iteration_bound: int
    iterations: int
    separated: bool
    reason: str


@dataclass
class SearchOut:
    lower: float
    upper: float
    best_value: float
    best_y: np.ndarray
    total_iterations: int
    search_steps: int
    termination: str
    steps: list = field(default_factory=list)


class _Bracket:
    """R/meta.py:576-653."""

    def __init__(self, L, U, is_max, on_primal, gain_floor):
        self.L, self.U, self.is_max = L, U, is_max
        self.on_primal, self.gain_floor = on_primal, gain_floor
        self.best_f = self.best_y = None

    def seed(self, f, y):
        self.best_f, self.best_y = f, np.asarray(y)
        self._certify(f)

    def _certify(self, f):
        if self.is_max:
            self.U = min(self.U, f)
        else:
            self.L = max(self.L, f)

    def absorb(self, res, alpha):
        before = self.U - self.L
        improved = False
        if isinstance(res, Primal):
            if self.is_max:
                self.L = max(self.L, alpha)
            else:
                self.U = min(self.U, alpha)
            if self.on_primal is not None:
                c = self.on_primal(res)
                if c is not None:
                    if self.is_max:
                        self.L = max(self.L, c)
                    else:
                        self.U = min(self.U, c)
        else:
            if self.is_max:
                self.U = min(self.U, res.value)
            else:
                self.L = max(self.L, res.value)
        if res.best_progress is not None:
            f, y = res.best_progress, res.best_y
            if self.best_f is None or (f < self.best_f if self.is_max else f > self.best_f):
                if self.best_f is not None and \
                        abs(self.best_f - f) > self.gain_floor * abs(self.best_f):
                    improved = True
                self.best_f, self.best_y = f, y
            self._certify(self.best_f)
        if res.best_counter is not None:
            if self.is_max:
                self.L = max(self.L, res.best_counter)
            else:
                self.U = min(self.U, res.best_counter)
        return improved or (self.U - self.L) < before * (1.0 - 2e-2)

    def converged(self, eps):
        span = self.U - self.L
        ref = self.L if self.L > 0.0 else (span / 3.0 if self.is_max else 2.0 * span / 3.0)
        return span < eps * ref


def search(factory, L0, U0, eps, delta=1e-4, patience=10, enabled=True, progress=None,
           cap=None, seed=None, on_primal=None, zero_floor=None,
           refine_horizon=REFINE_HORIZON):
    """adaptive_search restated (R/meta.py:656-781)."""
    if not 0.0 <= L0 < U0:
        raise ValueError(f"need 0 <= L0 < U0, got [{L0}, {U0}]")
    if not 0.0 < eps < 1.0:
        raise ValueError("eps must be in (0, 1)")
    is_max = factory((L0 + U0) / 2.0).is_max
    br = _Bracket(float(L0), float(U0), is_max, on_primal, max(delta, eps / 10.0))
    if seed is not None:
        br.seed(*seed)
    total, steps = 0, []
    capped = floored = False
    test_cap = min(BRACKET_TEST_CAP, cap) if cap is not None else BRACKET_TEST_CAP
    while len(steps) < MAX_SEARCH_STEPS:
        if br.converged(eps):
            break
        span = br.U - br.L
        if zero_floor is not None and br.L == 0.0 and span < zero_floor:
            floored = True
            break
        alpha = br.L + span / 3.0 if is_max else br.L + 2.0 * span / 3.0
        eps_i = span / (3.0 * alpha)
        spec = factory(alpha)
        T_i = iteration_bound(spec.R, spec.rho, spec.rank, eps_i, alpha)
        res = ftp(spec, alpha, eps_i, delta, patience, enabled, progress, test_cap)
        total += res.iterations
        if cap is not None and cap < T_i and isinstance(res, Dual) \
                and res.reason == "exhausted" and res.iterations >= cap:
            capped = True
        productive = br.absorb(res, alpha)
        steps.append(StepRec(alpha, eps_i, T_i, res.iterations, isinstance(res, Primal),
                             getattr(res, "reason", "separated")))
        if not productive:
            break
    if progress is not None and not floored:
        h = REFINE_START
        for _ in range(MAX_REFINE_ROUNDS):
            if br.converged(eps) or len(steps) >= MAX_SEARCH_STEPS:
                break
            alpha = (br.L + br.U) / 2.0
            if alpha <= 0.0:
                break
            spec = factory(alpha)
            T_i = iteration_bound(spec.R, spec.rho, spec.rank, eps, alpha)
            full = min(T_i, refine_horizon, cap) if cap is not None \
                else min(T_i, refine_horizon)
            horizon = min(h, full)
            res = refine(spec, alpha, horizon, delta, patience, enabled, progress,
                         max(delta, eps / 20.0), (br.L, br.U), eps)
            total += res.iterations
            productive = br.absorb(res, alpha)
            steps.append(StepRec(alpha, eps, T_i, res.iterations, isinstance(res, Primal),
                                 getattr(res, "reason", "separated")))
            if not productive and horizon >= full:
                break
            h = min(h * 4, refine_horizon)
    if br.best_f is None or br.best_y is None:
        raise RuntimeError("search finished without any certified solution")
    term = ("IterationCap" if capped else
            "RangeConverged" if br.converged(eps) else "EarlyStopped")
    return SearchOut(br.L, br.U, br.best_f, br.best_y, total, len(steps), term, steps)


# ------------------------------------------------------------------ solvers
def solve_ses(centers, radii, eps, delta=1e-4, patience=10, threads=1, cap=None,
              early_stop=True):
    """solve_ses restated (R/ses.py:135-194). Returns a dict."""
    prob = SesProblem(centers, radii, max(1, int(threads)))
    D, L0, U0 = prob.range()
    d = prob.d
    if D == 0.0:
        return {"radius": 0.0, "center": prob.c[0].copy(), "slack": 0.0, "primal": 0.0,
                "iterations": 0, "steps": 0, "termination": "RangeConverged",
                "search": []}
    rho = 3.0 * D / SQRT2
    spec = prob.spec(rho)
    v1 = prob.c[0]
    f0 = prob.progress(v1)
    out = search(lambda a: spec, L0, U0, eps, delta, patience, early_stop,
                 lambda y: prob.progress(y[:d]), cap, (f0, np.concatenate([v1, [f0]])))
    center = out.best_y[:d].copy()
    radius = out.best_value
    return {"radius": radius, "center": center, "slack": prob.progress(center) - radius,
            "primal": out.lower, "iterations": out.total_iterations,
            "steps": out.search_steps, "termination": out.termination,
            "search": out.steps}


def solve_svm(P, Q, eps, delta=1e-4, patience=10, threads=1, cap=None, early_stop=True):
    """solve_svm restated (R/svm.py:153-246). Returns a dict."""
    prob = SvmProblem(P, Q, max(1, int(threads)))
    D, d = prob.D, prob.d
    spec = prob.spec()
    w0 = prob.P.mean(axis=0) - prob.Q.mean(axis=0)
    if np.linalg.norm(w0) == 0.0:
        w0 = np.zeros(d)
        w0[0] = 1.0
    f0 = prob.progress(w0)
    out = search(lambda a: spec, 0.0, 2.0 * D, SVM_SEARCH_EPS_FACTOR * eps, delta,
                 patience, early_stop, lambda y: prob.progress(y[:d]), cap,
                 (f0, np.concatenate([w0, [0.0, 0.0]])),
                 on_primal=lambda c: prob.counter(c.p)[0],
                 zero_floor=SVM_INFEASIBLE_FLOOR * 2.0 * D)
    if out.lower == 0.0 and out.upper <= SVM_INFEASIBLE_FLOOR * 2.0 * D:
        raise RuntimeError("InfeasibleInput: certified margin stayed zero")
    w_raw = out.best_y[:d]
    wn = float(np.linalg.norm(w_raw))
    if wn > 0.0:
        w = w_raw / wn
    else:
        w = np.zeros(d)
        w[0] = 1.0
    if prob.best_dist is not None:
        mu, gam = prob.best_pair
        dist = prob.best_dist
    else:
        mu = np.full(prob.n1, 1.0 / prob.n1)
        gam = np.full(prob.n2, 1.0 / prob.n2)
        dist = float(np.linalg.norm(prob.P.T @ mu - prob.Q.T @ gam))
    proxy = dist if dist > 0.0 else 1.0
    return {"margin": out.best_value, "w": w, "mu": mu, "gam": gam, "pd_distance": dist,
            "excentricity": (D / proxy) ** 2, "primal": out.best_value,
            "iterations": out.total_iterations, "steps": out.search_steps,
            "termination": out.termination, "search": out.steps}


# ------------------------------------------------------------------ instance generators
def gen_ses(n, d, seed, dist="gaussian"):
    """R/instances.py:155-175 (same generator call sequence)."""
    rng = np.random.default_rng(seed)
    if dist == "gaussian":
        pts = rng.standard_normal((n, d))
    elif dist == "uniform-ball":
        dirs = rng.standard_normal((n, d))
        dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
        pts = dirs * rng.random(n)[:, None] ** (1.0 / d)
    elif dist == "sphere-surface":
        k = n // 2
        dirs = rng.standard_normal((k + n % 2, d))
        dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
        pts = np.concatenate([dirs[:k], -dirs[:k], dirs[k:]])
    else:
        raise ValueError(dist)
    return pts, np.zeros(n)


def gen_svm(n1, n2, d, seed, gap=1.0):
    """R/instances.py:178-199."""
    rng = np.random.default_rng(seed)
    direction = rng.standard_normal(d)
    direction /= np.linalg.norm(direction)
    off = (1.0 + gap / 2.0) * direction

    def ball(k):
        dirs = rng.standard_normal((k, d))
        dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
        return dirs * rng.random(k)[:, None] ** (1.0 / d)

    P = ball(n1) + off
    Q = ball(n2) - off
    return P, Q, direction
