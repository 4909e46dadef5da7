"""ctypes binding of the C ABI in include/scmwu.h.

The product loads ``libscmwu.so`` (built in-tree by ``build.py`` / ``__graft_entry__.build()``)
from this package directory.  There is no CPU fallback: if the library is
missing, or reports that no CUDA device is usable, the solvers raise.
"""
from __future__ import annotations

import ctypes
import math
import os
from typing import Optional

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_NAME = "libscmwu.so"

SC_OK, SC_EARG, SC_ECUDA, SC_ENCCL, SC_EWIDTH, SC_EOOM, SC_ETRACE = range(7)
SC_SES, SC_SVM = 0, 1
SC_MODE_FTP, SC_MODE_REFINE = 0, 1
SC_PRIMAL, SC_DUAL = 0, 1
REASONS = {0: "separated", 1: "exhausted", 2: "early_stop", 3: "affirmative", 4: "refined"}

INT64_MAX = (1 << 63) - 1


class NativeUnavailable(RuntimeError):
    """The CUDA engine library is missing or cannot run here."""


class NativeError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        super().__init__(f"scmwu status {status}: {msg}")


class ScProblem(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("d", ctypes.c_int32), ("n", ctypes.c_int64),
                ("n1", ctypes.c_int64), ("D", ctypes.c_double), ("rho", ctypes.c_double),
                ("R", ctypes.c_double), ("rank", ctypes.c_int64), ("ln_r", ctypes.c_double),
                ("grid", ctypes.c_int32), ("device", ctypes.c_int32),
                ("world", ctypes.c_int32), ("shard", ctypes.c_int32), ("row0", ctypes.c_int64),
                ("n_local", ctypes.c_int64), ("n1_local", ctypes.c_int64)]


SC_GEN_GAUSSIAN, SC_GEN_UNIFORM_BALL, SC_GEN_SPHERE_SURFACE, SC_GEN_SVM_CLUSTERS = 0, 1, 2, 3
GEN_DISTS = {"gaussian": SC_GEN_GAUSSIAN, "uniform-ball": SC_GEN_UNIFORM_BALL,
             "sphere-surface": SC_GEN_SPHERE_SURFACE}


class ScGen(ctypes.Structure):
    _fields_ = [("dist", ctypes.c_int32), ("seed", ctypes.c_uint64), ("gap", ctypes.c_double),
                ("direction", ctypes.POINTER(ctypes.c_double))]


class ScFtpArgs(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("has_progress", ctypes.c_int32),
                ("alpha", ctypes.c_double), ("eps", ctypes.c_double),
                ("budget", ctypes.c_int64), ("horizon", ctypes.c_int64),
                ("ceil_ln_r", ctypes.c_int64), ("delta", ctypes.c_double),
                ("patience", ctypes.c_int32), ("enabled", ctypes.c_int32),
                ("gain_rel", ctypes.c_double), ("lo", ctypes.c_double),
                ("hi", ctypes.c_double), ("target", ctypes.c_double)]


class ScFtpResult(ctypes.Structure):
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


class ScSolveArgs(ctypes.Structure):
    _fields_ = [("eps", ctypes.c_double), ("L0", ctypes.c_double), ("U0", ctypes.c_double),
                ("delta", ctypes.c_double), ("patience", ctypes.c_int32),
                ("enabled", ctypes.c_int32), ("cap", ctypes.c_int64),
                ("ceil_ln_r", ctypes.c_int64), ("refine_horizon", ctypes.c_int64),
                ("zero_lower_floor", ctypes.c_double), ("on_primal", ctypes.c_int32),
                ("max_steps", ctypes.c_int32)]


class ScSearchStep(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_double), ("eps", ctypes.c_double),
                ("iteration_bound", ctypes.c_int64), ("iterations", ctypes.c_int64),
                ("separated", ctypes.c_int32), ("reason", ctypes.c_int32)]


class ScSolveResult(ctypes.Structure):
    _fields_ = [("lower", ctypes.c_double), ("upper", ctypes.c_double),
                ("best_value", ctypes.c_double), ("has_best", ctypes.c_int32),
                ("termination", ctypes.c_int32), ("total_iterations", ctypes.c_int64),
                ("search_steps", ctypes.c_int32), ("has_pd", ctypes.c_int32),
                ("pd_dist", ctypes.c_double), ("seed_f", ctypes.c_double),
                ("final_f", ctypes.c_double), ("width_alpha", ctypes.c_double),
                ("width_iteration", ctypes.c_int64), ("width_norm", ctypes.c_double),
                ("passes", ctypes.c_int64), ("kernel_ms", ctypes.c_float),
                ("width_passes", ctypes.c_int64)]


SC_TERMINATIONS = {0: "IterationCap", 1: "RangeConverged", 2: "EarlyStopped"}
MAX_SEARCH_STEPS = 400

EXPORTS = ("sc_create", "sc_ftp", "sc_progress", "sc_iterate", "sc_pd_commit", "sc_pd_pair",
           "sc_set_grid", "sc_info", "sc_mark", "sc_elapsed", "sc_launches", "sc_debug_timing",
           "sc_local_red0", "sc_progress_parts", "sc_set_globals", "sc_ipc_handle",
           "sc_connect", "sc_last_error", "sc_destroy", "sc_version", "sc_create_generated",
           "sc_set_range", "sc_read_rows", "sc_meb_baseline", "sc_gilbert_baseline",
           "sc_pool_trim", "sc_solve", "sc_row_range")

_dp = ctypes.POINTER(ctypes.c_double)


def _ptr(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(_dp)


class Engine:
    """One loaded implementation of the C ABI."""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} is missing: build it with `python build.py` "
                f"(nvcc, sm_100a); there is no CPU fallback")
        self.path = path
        lib = ctypes.CDLL(path)
        vp = ctypes.c_void_p
        lib.sc_create.argtypes = [ctypes.POINTER(ScProblem), _dp, _dp, _dp, ctypes.POINTER(vp)]
        lib.sc_ftp.argtypes = [vp, ctypes.POINTER(ScFtpArgs), ctypes.POINTER(ScFtpResult), _dp,
                               _dp]
        lib.sc_progress.argtypes = [vp, _dp, _dp]
        lib.sc_iterate.argtypes = [vp, _dp]
        lib.sc_pd_commit.argtypes = [vp, ctypes.c_int32]
        lib.sc_pd_pair.argtypes = [vp, _dp, _dp, _dp]
        lib.sc_set_grid.argtypes = [vp, ctypes.c_int32]
        lib.sc_info.argtypes = [vp, ctypes.POINTER(ctypes.c_int64)]
        lib.sc_last_error.argtypes = [vp]
        lib.sc_last_error.restype = ctypes.c_char_p
        lib.sc_destroy.argtypes = [vp]
        lib.sc_destroy.restype = None
        lib.sc_version.restype = ctypes.c_int
        lib.sc_pool_trim.argtypes = [ctypes.c_int32]
        lib.sc_solve.argtypes = [vp, ctypes.POINTER(ScSolveArgs), _dp,
                                 ctypes.POINTER(ScSolveResult), _dp,
                                 ctypes.POINTER(ScSearchStep)]
        lib.sc_mark.argtypes = [vp, ctypes.c_int32]
        lib.sc_elapsed.argtypes = [vp, ctypes.POINTER(ctypes.c_float)]
        lib.sc_launches.argtypes = [vp]
        lib.sc_launches.restype = ctypes.c_int64
        lib.sc_debug_timing.argtypes = [vp, _dp]
        lib.sc_local_red0.argtypes = [vp, _dp]
        lib.sc_progress_parts.argtypes = [vp, _dp, _dp]
        lib.sc_set_globals.argtypes = [vp, _dp, _dp, ctypes.c_double]
        lib.sc_ipc_handle.argtypes = [vp, ctypes.c_char_p]
        lib.sc_connect.argtypes = [vp, ctypes.c_char_p]
        lib.sc_create_generated.argtypes = [ctypes.POINTER(ScProblem), ctypes.POINTER(ScGen),
                                            _dp, ctypes.POINTER(vp)]
        lib.sc_set_range.argtypes = [vp, ctypes.c_double]
        lib.sc_row_range.argtypes = [vp, _dp]
        lib.sc_read_rows.argtypes = [vp, ctypes.c_int64, ctypes.c_int64, _dp]
        lib.sc_meb_baseline.argtypes = [vp, ctypes.c_int64, _dp, _dp]
        lib.sc_gilbert_baseline.argtypes = [vp, ctypes.c_double, ctypes.c_int64, _dp, _dp,
                                            ctypes.POINTER(ctypes.c_int64), _dp, _dp]
        self.lib = lib

    def trim_pool(self, device: int = 0) -> None:
        """Return the device memory the engine's private pool keeps for reuse
        (sc_pool_trim)."""
        st = self.lib.sc_pool_trim(device)
        if st != SC_OK:
            raise RuntimeError(f"sc_pool_trim failed with status {st}")

    def create_generated(self, kind: int, n: int, d: int, seed: int, dist: int,
                         n1: int = 0, gap: float = 1.0, direction=None, grid: int = 0,
                         device: int = 0, shard: Optional[tuple] = None
                         ) -> tuple["Handle", float, Optional[np.ndarray]]:
        """Draw the instance on the device (sc_create_generated).  ``shard = (world, index,
        row0, n_local)``.  Returns (handle, this shard's range D, SES anchor row v1)."""
        world, index, row0, n_local = 1, 0, 0, n
        if shard is not None and shard[0] > 1:
            world, index, row0, n_local = shard
        n1_local = max(0, min(n_local, n1 - row0)) if kind == SC_SVM else 0
        prob = ScProblem(kind=kind, d=d, n=n, n1=n1, grid=grid, device=device, world=world,
                         shard=index, row0=row0, n_local=n_local, n1_local=n1_local)
        dvec = None
        if direction is not None:
            dvec = np.ascontiguousarray(direction, dtype=np.float64)
        gen = ScGen(dist=dist, seed=seed, gap=gap, direction=_ptr(dvec))
        v1 = np.zeros(d) if kind == SC_SES else None
        h = ctypes.c_void_p()
        st = self.lib.sc_create_generated(ctypes.byref(prob), ctypes.byref(gen), _ptr(v1),
                                          ctypes.byref(h))
        if st != SC_OK:
            msg = self.lib.sc_last_error(h).decode() if h.value else "sc_create_generated failed"
            if h.value:
                self.lib.sc_destroy(h)
            if st == SC_ECUDA:
                raise NativeUnavailable(f"CUDA engine cannot run: {msg}")
            raise NativeError(st, msg)
        return Handle(self, h, prob), float(prob.D), v1

    def create(self, kind: int, X, X_tail, radii, D: float, rho: float, R: float,
               rank: int, n1: int = 0, grid: int = 0, device: int = 0,
               shard: Optional[tuple] = None) -> "Handle":
        """``shard = (world, index, row0, n_global)``: X holds rows [row0, row0 + len(X))
        of an n_global-row matrix (one GPU of a row-sharded solve)."""
        X = np.ascontiguousarray(X, dtype=np.float64)
        Xt = None if X_tail is None else np.ascontiguousarray(X_tail, dtype=np.float64)
        rad = None if radii is None else np.ascontiguousarray(radii, dtype=np.float64)
        n = X.shape[0] + (0 if Xt is None else Xt.shape[0])
        d = X.shape[1]
        world, index, row0, n_local = 1, 0, 0, n
        if shard is not None and shard[0] > 1:
            world, index, row0, n = shard
        n1_local = max(0, min(n_local, n1 - row0)) if kind == SC_SVM else 0
        prob = ScProblem(kind=kind, d=d, n=n, n1=n1, D=D, rho=rho, R=R, rank=rank,
                         ln_r=math.log(rank), grid=grid, device=device, world=world,
                         shard=index, row0=row0, n_local=n_local, n1_local=n1_local)
        h = ctypes.c_void_p()
        st = self.lib.sc_create(ctypes.byref(prob), _ptr(X), _ptr(Xt), _ptr(rad),
                                ctypes.byref(h))
        if st != SC_OK:
            msg = self.lib.sc_last_error(h).decode() if h.value else "sc_create failed"
            if h.value:
                self.lib.sc_destroy(h)
            if st == SC_ECUDA:
                raise NativeUnavailable(f"CUDA engine cannot run: {msg}")
            raise NativeError(st, msg)
        return Handle(self, h, prob)


class FtpOut:
    """Plain view of one sc_ftp call."""

    __slots__ = ("status", "kind", "reason", "iterations", "eps_eff", "value", "oracle_value",
                 "best_f", "best_counter", "y_tilde", "best_y", "width_iteration",
                 "width_norm", "counter_min", "sep_dist", "passes", "kernel_ms", "has_claim_y",
                 "width_passes")


class Handle:
    def __init__(self, engine: Engine, h: ctypes.c_void_p, prob: ScProblem):
        self.engine = engine
        self.h = h
        self.prob = prob
        self.d = prob.d
        self.dual_dim = prob.d + (1 if prob.kind == SC_SES else 2)
        self.calls = 0

    def _check(self, st: int, what: str):
        if st != SC_OK:
            raise NativeError(st, f"{what}: {self.engine.lib.sc_last_error(self.h).decode()}")

    def ftp(self, args: ScFtpArgs) -> FtpOut:
        res = ScFtpResult()
        yt = np.zeros(self.dual_dim)
        by = np.zeros(self.dual_dim)
        st = self.engine.lib.sc_ftp(self.h, ctypes.byref(args), ctypes.byref(res), _ptr(yt),
                                    _ptr(by))
        self.calls += 1
        if st not in (SC_OK, SC_EWIDTH):
            self._check(st, "sc_ftp")
        o = FtpOut()
        o.status = st
        o.kind = res.kind
        o.reason = REASONS.get(res.reason, "?")
        o.iterations = int(res.iterations)
        o.eps_eff = res.eps_eff
        o.value = res.value
        o.oracle_value = res.oracle_value
        o.best_f = res.best_f if res.has_best_f else None
        o.best_counter = res.best_counter if res.has_best_counter else None
        o.y_tilde = yt
        o.best_y = by if res.has_best_f else None
        o.has_claim_y = bool(res.has_claim_y)
        o.width_iteration = int(res.width_iteration)
        o.width_norm = res.width_norm
        o.counter_min = res.counter_min if res.has_counter_min else None
        o.sep_dist = res.sep_dist
        o.passes = int(res.passes)
        o.kernel_ms = float(res.kernel_ms)
        o.width_passes = int(res.width_passes)
        return o

    def solve(self, args: ScSolveArgs, seed_y):
        """A whole adaptive search in one launch (sc_solve).  Returns (status, result,
        best_y, steps)."""
        seed = np.ascontiguousarray(np.asarray(seed_y, dtype=np.float64)[: self.d])
        res = ScSolveResult()
        by = np.zeros(self.dual_dim)
        steps = (ScSearchStep * max(1, args.max_steps))()
        st = self.engine.lib.sc_solve(self.h, ctypes.byref(args), _ptr(seed), ctypes.byref(res),
                                      _ptr(by), steps)
        self.calls += 1
        if st not in (SC_OK, SC_EWIDTH):
            self._check(st, "sc_solve")
        return st, res, by, [steps[i] for i in range(min(res.search_steps, args.max_steps))]

    def progress(self, y) -> float:
        y = np.ascontiguousarray(np.asarray(y, dtype=np.float64)[: self.d])
        f = ctypes.c_double()
        self._check(self.engine.lib.sc_progress(self.h, _ptr(y), ctypes.byref(f)), "sc_progress")
        return float(f.value)

    def iterate(self) -> np.ndarray:
        """p of the last call over this handle's rows (sharded: the local block)."""
        n, d = self.prob.n_local, self.prob.d
        first = 1 if self.prob.kind == SC_SES and self.prob.row0 == 0 else 0
        size = (n - first) * (d + 1) if self.prob.kind == SC_SES else n
        out = np.empty(size)
        self._check(self.engine.lib.sc_iterate(self.h, _ptr(out)), "sc_iterate")
        return out

    def pd_commit(self, which: int) -> None:
        self._check(self.engine.lib.sc_pd_commit(self.h, which), "sc_pd_commit")

    def pd_pair(self):
        """(mu, gam, dist) for this handle's rows; sharded handles return the raw
        local weights (dist NaN) and the caller normalises across ranks."""
        n1 = self.prob.n1_local
        mu = np.empty(n1)
        gam = np.empty(self.prob.n_local - n1)
        dist = ctypes.c_double()
        self._check(self.engine.lib.sc_pd_pair(self.h, _ptr(mu), _ptr(gam), ctypes.byref(dist)),
                    "sc_pd_pair")
        return mu, gam, float(dist.value)

    # ---- row sharding
    def local_red0(self) -> np.ndarray:
        rw = self.prob.d + (7 if self.prob.kind == SC_SES else 12 + self.prob.d)
        out = np.zeros(rw)
        self._check(self.engine.lib.sc_local_red0(self.h, _ptr(out)), "sc_local_red0")
        return out

    def set_globals(self, red0, v1=None, g1: float = 0.0) -> None:
        red0 = np.ascontiguousarray(red0, dtype=np.float64)
        v = None if v1 is None else np.ascontiguousarray(v1, dtype=np.float64)
        self._check(self.engine.lib.sc_set_globals(self.h, _ptr(red0), _ptr(v), g1),
                    "sc_set_globals")

    def set_range(self, D: float) -> None:
        self._check(self.engine.lib.sc_set_range(self.h, D), "sc_set_range")
        # the constants the library derived (R/ses.py:161,169, R/svm.py:168,186)
        p = self.prob
        p.D = D
        if p.kind == SC_SES:
            p.rho, p.R, p.rank = 3.0 * D / math.sqrt(2.0), math.sqrt(2.0), 2 * (p.n - 1)
        else:
            p.rho, p.R, p.rank = 2.0 * D, 2.0, p.n
        p.ln_r = math.log(p.rank)

    def row_range(self) -> float:
        """The reference's range expression over this handle's rows, evaluated on the
        device in numpy's operation order (sc_row_range): bit-identical to ses_range /
        max_norm over the same rows; -inf for a shard without such rows."""
        D = ctypes.c_double()
        self._check(self.engine.lib.sc_row_range(self.h, ctypes.byref(D)), "sc_row_range")
        return float(D.value)

    def set_range_from_rows(self) -> float:
        """D of a single-GPU handle from its resident rows, then sc_set_range."""
        D = self.row_range()
        self.set_range(D)
        return D

    def meb_baseline(self, iters: int) -> tuple[np.ndarray, float]:
        c = np.zeros(self.d)
        v = ctypes.c_double()
        self._check(self.engine.lib.sc_meb_baseline(self.h, iters, _ptr(c), ctypes.byref(v)),
                    "sc_meb_baseline")
        return c, float(v.value)

    def gilbert_baseline(self, gap_tol: float, max_iters: int, weights: bool = True):
        n1 = self.prob.n1_local
        n2 = self.prob.n_local - n1
        mu = np.zeros(n1) if weights else None
        gam = np.zeros(n2) if weights else None
        v, g, it = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        self._check(self.engine.lib.sc_gilbert_baseline(
            self.h, gap_tol, max_iters, ctypes.byref(v), ctypes.byref(g), ctypes.byref(it),
            _ptr(mu), _ptr(gam)), "sc_gilbert_baseline")
        return float(v.value), float(g.value), int(it.value), mu, gam

    def read_rows(self, first: int = 0, count: Optional[int] = None) -> np.ndarray:
        if count is None:
            count = self.prob.n_local - first
        out = np.zeros((count, self.d))
        self._check(self.engine.lib.sc_read_rows(self.h, first, count, _ptr(out)),
                    "sc_read_rows")
        return out

    def progress_parts(self, y) -> np.ndarray:
        y = np.ascontiguousarray(np.asarray(y, dtype=np.float64)[: self.d])
        out = np.zeros(2)
        self._check(self.engine.lib.sc_progress_parts(self.h, _ptr(y), _ptr(out)),
                    "sc_progress_parts")
        return out

    def ipc_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        self._check(self.engine.lib.sc_ipc_handle(self.h, buf), "sc_ipc_handle")
        return buf.raw

    def connect(self, handles: list) -> None:
        blob = b"".join(handles)
        self._check(self.engine.lib.sc_connect(self.h, blob), "sc_connect")

    def pd_reset(self) -> None:
        self._check(self.engine.lib.sc_pd_commit(self.h, 2), "sc_pd_commit")

    def mark(self, which: int) -> None:
        self._check(self.engine.lib.sc_mark(self.h, which), "sc_mark")

    def elapsed_ms(self) -> float:
        ms = ctypes.c_float()
        self._check(self.engine.lib.sc_elapsed(self.h, ctypes.byref(ms)), "sc_elapsed")
        return float(ms.value)

    def debug_timing(self) -> np.ndarray:
        """[0:9] phase cycles of CTA 0, [9:169] per-CTA streaming cycles, [169:329] SM ids,
        [329:489] / [489:649] global-ns start / end of each CTA's last streaming pass,
        [649:809] / [809:969] global-ns arrival at / release from its first grid barrier,
        [969:976] cycle sums of the control tail's sections (CTA 0)."""
        out = np.zeros(9 + 6 * 160 + 7)
        self._check(self.engine.lib.sc_debug_timing(self.h, _ptr(out)), "sc_debug_timing")
        return out

    def launches(self) -> int:
        return int(self.engine.lib.sc_launches(self.h))

    def set_grid(self, grid: int) -> None:
        self._check(self.engine.lib.sc_set_grid(self.h, grid), "sc_set_grid")

    def info(self) -> dict:
        out = (ctypes.c_int64 * 8)()
        self._check(self.engine.lib.sc_info(self.h, out), "sc_info")
        keys = ("grid", "threads", "lanes_per_row", "cols_per_lane", "tile_rows", "stages",
                "resident", "smem_bytes")
        return dict(zip(keys, [int(v) for v in out]))

    def close(self) -> None:
        if self.h is not None and self.h.value:
            self.engine.lib.sc_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


_cuda_engine: Optional[Engine] = None


def cuda_engine() -> Engine:
    """The B200 engine (paper_2405_09157_b200/libscmwu.so).  Raises if absent."""
    global _cuda_engine
    if _cuda_engine is None:
        # SCMWU_LIB: an alternative build of the same CUDA engine (A/B performance runs)
        _cuda_engine = Engine(os.environ.get("SCMWU_LIB") or os.path.join(PKG_DIR, LIB_NAME))
    return _cuda_engine
