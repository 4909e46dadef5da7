"""Row sharding of one solve across GPUs — one process per GPU.

Rows are split into contiguous ranges (the partition of ``np.array_split``,
like the reference's ``_reduce.part_sum``, R/_reduce.py:12-26).  Every rank
holds one range in its HBM and runs the SAME host control (adaptive search)
on identical results, because the per-pass reduction is exchanged inside the
persistent kernel: each rank writes its folded pass vector into every peer's
mailbox over NVLink (CUDA IPC mappings, exchanged once here) and all ranks
fold the rank vectors in rank order.  Host-side one-off quantities (the
iterate-1 sums, progress extremes, the polytope-distance pair) are combined
here through ``torch.distributed`` with the same rank-ordered fold.

With the CPU emulator (tests only) the in-kernel exchange is replaced by a
callback that performs the same fold over a gloo all-gather.
"""
from __future__ import annotations

import ctypes
import math
from typing import Optional

import numpy as np

from . import _native as nat
from .cones import SQRT2
from .meta import DeviceProblem

# combine operator of every reduced column (mirror of red_op in scmwu_kernel.cuh)
_SUM, _MAX, _MIN = 0, 1, 2


def red_ops(kind: int, d: int) -> np.ndarray:
    if kind == nat.SC_SES:
        ops = np.zeros(7 + d, dtype=np.int64)
        ops[[3, 4, 5, 6]] = _MAX
    else:
        ops = np.zeros(12 + 2 * d, dtype=np.int64)
        ops[[2, 5, 7, 9, 11]] = _MAX
        ops[[3, 4, 6, 8, 10]] = _MIN
    return ops


def fold_ranks(rows: np.ndarray, ops: np.ndarray) -> np.ndarray:
    """Fold rank vectors in rank order: acc = op(acc, v_r) from the identity."""
    acc = np.where(ops == _SUM, 0.0, np.where(ops == _MAX, -np.inf, np.inf))
    for v in rows:
        acc = np.where(ops == _SUM, acc + v, np.where(ops == _MAX, np.fmax(acc, v),
                                                     np.fmin(acc, v)))
    return acc


def row_ranges(n: int, world: int) -> list[tuple[int, int]]:
    """np.array_split boundaries: the first n % world ranges get one extra row."""
    if world < 1 or n < world:
        raise ValueError(f"cannot split {n} rows over {world} ranks")
    base, extra = divmod(n, world)
    out, a = [], 0
    for r in range(world):
        b = a + base + (1 if r < extra else 0)
        out.append((a, b))
        a = b
    return out


class Comm:
    """The few host collectives a sharded solve needs, over torch.distributed."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_gather_array(self, a: np.ndarray) -> np.ndarray:
        import torch
        backend = self.dist.get_backend(self.group)
        dev = "cuda" if backend == "nccl" else "cpu"
        t = torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)
        outs = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(outs, t, group=self.group)
        return np.stack([o.cpu().numpy() for o in outs])

    def all_gather_object(self, obj) -> list:
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out


class ShardedDeviceProblem(DeviceProblem):
    """A DeviceProblem over this rank's rows; progress / pair are folded across ranks."""

    def __init__(self, handle: nat.Handle, cone, kind: int, comm: Comm):
        super().__init__(handle, cone, kind)
        self.comm = comm
        self._cb = None

    def progress(self, y_bar) -> float:
        y = np.asarray(y_bar, dtype=np.float64)
        parts = self.comm.all_gather_array(self.handle.progress_parts(y))
        if self.kind == nat.SC_SES:
            return float(np.max(parts[:, 0]))
        minP, maxQ = float(np.min(parts[:, 0])), float(np.max(parts[:, 1]))
        nrm = float(math.sqrt(float(np.dot(y[: self.handle.d], y[: self.handle.d]))))
        if nrm == 0.0:
            return 0.0
        sep = (minP - maxQ) / nrm
        return sep if sep > 0.0 else 0.0

    def pd_pair(self):
        mu_l, gam_l, _ = self.handle.pd_pair()   # raw local weights
        sums = self.comm.all_gather_array(np.array([mu_l.sum(), gam_l.sum()]))
        sP, sQ = 0.0, 0.0
        for s in sums:        # rank order
            sP += s[0]
            sQ += s[1]
        parts = self.comm.all_gather_object((mu_l / sP, gam_l / sQ))
        mu = np.concatenate([p[0] for p in parts])
        gam = np.concatenate([p[1] for p in parts])
        dist = self.best_pd_dist if self.best_pd_dist is not None else float("nan")
        return mu, gam, dist


def _connect(h: nat.Handle, comm: Comm, kind: int, d: int, dev: ShardedDeviceProblem):
    emu_hook = getattr(h.engine.lib, "emu_set_exchange", None)
    if emu_hook is None:
        # CUDA: map every rank's mailbox (the exchange then runs inside the kernel)
        h.connect(comm.all_gather_object(h.ipc_handle()))
        return
    ops = red_ops(kind, d)
    cbtype = ctypes.CFUNCTYPE(None, ctypes.POINTER(ctypes.c_double), ctypes.c_int,
                              ctypes.POINTER(ctypes.c_double))

    def exchange(local, rw, out):
        loc = np.ctypeslib.as_array(local, shape=(rw,)).copy()
        red = fold_ranks(comm.all_gather_array(loc), ops)
        np.ctypeslib.as_array(out, shape=(rw,))[:] = red

    dev._cb = cbtype(exchange)          # keep the callback alive with the problem
    emu_hook.argtypes = [ctypes.c_void_p, cbtype]
    emu_hook(h.h, dev._cb)


def _global_max(comm: Comm, x: float) -> float:
    return float(np.max(comm.all_gather_array(np.array([x]))))


def ses_device_sharded(inst, comm: Comm, engine: Optional[nat.Engine] = None, device: int = 0,
                       grid: int = 0) -> ShardedDeviceProblem:
    """This rank's share of an SES instance (every rank passes the full instance, e.g. a
    memory map; only this rank's rows are read and uploaded).  The range D is the
    reference's expression (R/ses.py:65-72) over this rank's resident rows (sc_row_range,
    numpy's operation order), max-reduced across ranks: bit-identical to the
    single-process value."""
    from .ses import ses_cone
    eng = engine if engine is not None else nat.cuda_engine()
    n = inst.n
    r0, r1 = row_ranges(n, comm.world)[comm.rank]
    h = eng.create(nat.SC_SES, inst.centers[r0:r1], None, inst.radii[r0:r1], D=0.0,
                   rho=0.0, R=SQRT2, rank=2 * (n - 1), grid=grid, device=device,
                   shard=(comm.world, comm.rank, r0, n))
    ops = red_ops(nat.SC_SES, inst.d)
    h.set_globals(fold_ranks(comm.all_gather_array(h.local_red0()), ops), inst.centers[0],
                  float(inst.radii[0]))
    h.set_range(_global_max(comm, h.row_range()))   # needs v1 and g1 (set_globals)
    dev = ShardedDeviceProblem(h, ses_cone(n, inst.d), nat.SC_SES, comm)
    _connect(h, comm, nat.SC_SES, inst.d, dev)
    return dev


def svm_device_sharded(inst, comm: Comm, engine: Optional[nat.Engine] = None, device: int = 0,
                       grid: int = 0) -> ShardedDeviceProblem:
    """This rank's share of an SVM instance (rows P then Q, split contiguously)."""
    from .svm import svm_cone
    eng = engine if engine is not None else nat.cuda_engine()
    n1, n = inst.n1, inst.n1 + inst.n2
    r0, r1 = row_ranges(n, comm.world)[comm.rank]
    rows = np.concatenate([inst.P[max(r0, 0):min(r1, n1)],
                           inst.Q[max(r0 - n1, 0):max(r1 - n1, 0)]])
    h = eng.create(nat.SC_SVM, rows, None, None, D=0.0, rho=0.0, R=2.0, rank=n, n1=n1,
                   grid=grid, device=device, shard=(comm.world, comm.rank, r0, n))
    # max_norm (R/svm.py:62-66) over this rank's resident rows, max-reduced across ranks
    h.set_range(_global_max(comm, h.row_range()))
    ops = red_ops(nat.SC_SVM, inst.d)
    h.set_globals(fold_ranks(comm.all_gather_array(h.local_red0()), ops))
    dev = ShardedDeviceProblem(h, svm_cone(n), nat.SC_SVM, comm)
    _connect(h, comm, nat.SC_SVM, inst.d, dev)
    return dev
