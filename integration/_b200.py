"""symcone/_b200.py — ctypes binding of the B200 engine (libscmwu.so, include/scmwu.h)
for the reference package.  Dropped into symcone/ next to the patched meta.py, ses.py and
svm.py (integration/symcone_b200.patch); INTEGRATION.md §2-3 explains it.

Opt-in: the device path runs when SYMCONE_DEVICE=b200 (libscmwu.so from SCMWU_LIB, or the
repository build); otherwise the reference's own CPU loops run unchanged.  There is no
silent fallback: with the device requested, a missing library or GPU raises.
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

SC_SES, SC_SVM = 0, 1
SC_PRIMAL, SC_DUAL = 0, 1
SC_OK, SC_EARG, SC_ECUDA, SC_ENCCL, SC_EWIDTH, SC_EOOM = range(6)
_REASONS = {0: "separated", 1: "exhausted", 2: "early_stop", 3: "affirmative", 4: "refined"}
_dp, _vp = ctypes.POINTER(ctypes.c_double), ctypes.c_void_p


class Problem(ctypes.Structure):        # sc_problem
    _fields_ = [("kind", ctypes.c_int32), ("d", ctypes.c_int32), ("n", ctypes.c_int64),
                ("n1", ctypes.c_int64), ("D", ctypes.c_double), ("rho", ctypes.c_double),
                ("R", ctypes.c_double), ("rank", ctypes.c_int64), ("ln_r", ctypes.c_double),
                ("grid", ctypes.c_int32), ("device", ctypes.c_int32),
                ("world", ctypes.c_int32), ("shard", ctypes.c_int32), ("row0", ctypes.c_int64),
                ("n_local", ctypes.c_int64), ("n1_local", ctypes.c_int64)]


class Args(ctypes.Structure):           # sc_ftp_args
    _fields_ = [("mode", ctypes.c_int32), ("has_progress", ctypes.c_int32),
                ("alpha", ctypes.c_double), ("eps", ctypes.c_double),
                ("budget", ctypes.c_int64), ("horizon", ctypes.c_int64),
                ("ceil_ln_r", ctypes.c_int64), ("delta", ctypes.c_double),
                ("patience", ctypes.c_int32), ("enabled", ctypes.c_int32),
                ("gain_rel", ctypes.c_double), ("lo", ctypes.c_double),
                ("hi", ctypes.c_double), ("target", ctypes.c_double)]


class Result(ctypes.Structure):         # sc_ftp_result
    _fields_ = [("kind", ctypes.c_int32), ("reason", ctypes.c_int32),
                ("iterations", ctypes.c_int64), ("eps_eff", ctypes.c_double),
                ("value", ctypes.c_double), ("oracle_value", ctypes.c_double),
                ("has_best_f", ctypes.c_int32), ("has_best_counter", ctypes.c_int32),
                ("has_claim_y", ctypes.c_int32), ("best_f", ctypes.c_double),
                ("best_counter", ctypes.c_double), ("width_iteration", ctypes.c_int64),
                ("width_norm", ctypes.c_double), ("has_counter_min", ctypes.c_int32),
                ("counter_min", ctypes.c_double), ("sep_dist", ctypes.c_double),
                ("passes", ctypes.c_int64), ("kernel_ms", ctypes.c_float),
                ("width_passes", ctypes.c_int64)]


def enabled() -> bool:
    return os.environ.get("SYMCONE_DEVICE", "") == "b200"


_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.environ.get("SCMWU_LIB", "libscmwu.so")
        lib = ctypes.CDLL(path)
        lib.sc_create.argtypes = [ctypes.POINTER(Problem), _dp, _dp, _dp, ctypes.POINTER(_vp)]
        lib.sc_ftp.argtypes = [_vp, ctypes.POINTER(Args), ctypes.POINTER(Result), _dp, _dp]
        lib.sc_progress.argtypes = [_vp, _dp, _dp]
        lib.sc_pd_commit.argtypes = [_vp, ctypes.c_int32]
        lib.sc_pd_pair.argtypes = [_vp, _dp, _dp, _dp]
        lib.sc_last_error.argtypes = [_vp]
        lib.sc_last_error.restype = ctypes.c_char_p
        lib.sc_destroy.argtypes = [_vp]
        lib.sc_destroy.restype = None
        _LIB = lib
    return _LIB


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Device:
    """One application instance resident on the GPU (sc_create)."""

    def __init__(self, kind, X, X_tail, radii, D, rho, R, rank, n1=0):
        lib = _lib()
        X = _f64(X)
        Xt = None if X_tail is None else _f64(X_tail)
        rad = None if radii is None else _f64(radii)
        n = X.shape[0] + (0 if Xt is None else Xt.shape[0])
        self.kind, self.d, self.n, self.n1 = kind, X.shape[1], n, n1
        prob = Problem(kind=kind, d=self.d, n=n, n1=n1, D=D, rho=rho, R=R, rank=rank,
                       ln_r=math.log(rank))
        h = _vp()
        st = lib.sc_create(ctypes.byref(prob), X.ctypes.data_as(_dp),
                           None if Xt is None else Xt.ctypes.data_as(_dp),
                           None if rad is None else rad.ctypes.data_as(_dp), ctypes.byref(h))
        if st != SC_OK:
            msg = lib.sc_last_error(h).decode() if h.value else "sc_create failed"
            if h.value:
                lib.sc_destroy(h)
            raise RuntimeError(f"B200 engine: {msg} (status {st})")
        self.h = h
        self.best_pd = None          # best pd_counter distance committed on the device
        self.last_sep_dist = None    # pd_counter distance of the latest separation

    def close(self):
        if self.h is not None:
            _lib().sc_destroy(self.h)
            self.h = None

    def progress(self, y) -> float:
        y = _f64(y)
        f = ctypes.c_double()
        st = _lib().sc_progress(self.h, y.ctypes.data_as(_dp), ctypes.byref(f))
        if st != SC_OK:
            raise RuntimeError(f"sc_progress failed ({st})")
        return float(f.value)

    # ---- the two loop bodies of meta.py, one engine call each
    def _run(self, meta, oracle, alpha, args):
        dd = oracle.dual_dim
        res, yt, by = Result(), np.zeros(dd), np.zeros(dd)
        st = _lib().sc_ftp(self.h, ctypes.byref(args), ctypes.byref(res),
                           yt.ctypes.data_as(_dp), by.ctypes.data_as(_dp))
        if st == SC_EWIDTH:
            raise meta.WidthViolationError(alpha, oracle.width_rho, res.width_iteration,
                                           res.width_norm)
        if st == SC_EARG:
            raise ValueError(_lib().sc_last_error(self.h).decode())
        if st != SC_OK:
            raise RuntimeError(f"B200 engine: {_lib().sc_last_error(self.h).decode()}")
        # pd_counter side effect (svm.py best_pd): the call's smallest counter distance
        if self.kind == SC_SVM and res.has_counter_min and (
                self.best_pd is None or res.counter_min < self.best_pd):
            _lib().sc_pd_commit(self.h, 0)
            self.best_pd = res.counter_min
        best_f = res.best_f if res.has_best_f else None
        best_y = by.copy() if res.has_best_f else None
        best_c = res.best_counter if res.has_best_counter else None
        if res.kind == SC_PRIMAL:
            self.last_sep_dist = res.sep_dist
            return meta.PrimalCertificate(p=None, alpha=alpha, iterations=res.iterations,
                                          oracle_value=res.oracle_value, best_progress=best_f,
                                          best_y=best_y, best_counter=best_c)
        return meta.DualFeasible(y_tilde=yt, value=res.value, iterations=res.iterations,
                                 reason=_REASONS[res.reason], eps_eff=res.eps_eff,
                                 best_progress=best_f, best_y=best_y, best_counter=best_c,
                                 p_last=None)

    def solve_ftp(self, meta, oracle, alpha, eps, stopping, progress, cap):
        if alpha <= 0:
            raise ValueError("alpha must be positive")
        if eps <= 0:
            raise ValueError("eps must be positive")
        stopping = stopping or meta.EarlyStopConfig()
        budget = meta.iteration_bound(oracle.trace_bound, oracle.width_rho,
                                      oracle.cone.rank, eps, alpha)
        if cap is not None:
            budget = min(budget, cap)
        a = Args(mode=0, has_progress=int(progress is not None), alpha=alpha, eps=eps,
                 budget=min(budget, 1 << 62), horizon=0,
                 ceil_ln_r=math.ceil(math.log(oracle.cone.rank)), delta=stopping.delta,
                 patience=stopping.patience, enabled=int(stopping.enabled),
                 gain_rel=math.nan, lo=-math.inf, hi=math.inf, target=math.nan)
        return self._run(meta, oracle, alpha, a)

    def refine_run(self, meta, oracle, alpha, horizon, stopping, progress, gain_rel, bounds,
                   target):
        ln_r = math.log(oracle.cone.rank)
        lo, hi = bounds if bounds is not None else (-math.inf, math.inf)
        a = Args(mode=1, has_progress=int(progress is not None), alpha=alpha, eps=0.0,
                 budget=0, horizon=max(horizon, math.ceil(ln_r)), ceil_ln_r=math.ceil(ln_r),
                 delta=stopping.delta, patience=stopping.patience,
                 enabled=int(stopping.enabled),
                 gain_rel=stopping.delta if gain_rel is None else gain_rel, lo=lo, hi=hi,
                 target=math.nan if target is None else target)
        return self._run(meta, oracle, alpha, a)

    # ---- svm.py's pd_counter bookkeeping
    def on_primal(self, cert) -> float:
        """pd_counter(cert.p)[0] at the latest separation (svm.py on_primal)."""
        dist = self.last_sep_dist
        if self.best_pd is None or dist < self.best_pd:
            _lib().sc_pd_commit(self.h, 1)
            self.best_pd = dist
        return dist

    def best_pair(self):
        """(dist, (mu, gam)) of the best committed counter state, or (None, None)."""
        if self.best_pd is None:
            return None, None
        mu, gam = np.zeros(self.n1), np.zeros(self.n - self.n1)
        dist = ctypes.c_double()
        st = _lib().sc_pd_pair(self.h, mu.ctypes.data_as(_dp), gam.ctypes.data_as(_dp),
                               ctypes.byref(dist))
        if st != SC_OK:
            raise RuntimeError(f"sc_pd_pair failed ({st})")
        return self.best_pd, (mu, gam)


def ses_device(inst, D) -> Device:
    n = inst.n
    return Device(SC_SES, inst.centers, None, inst.radii, D, 3.0 * D / math.sqrt(2.0),
                  math.sqrt(2.0), 2 * (n - 1))


def svm_device(inst) -> Device:
    D = inst.max_norm
    return Device(SC_SVM, inst.P, inst.Q, None, D, 2.0 * D, 2.0, inst.n1 + inst.n2,
                  n1=inst.n1)
