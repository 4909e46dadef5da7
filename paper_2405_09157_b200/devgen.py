"""Instances that live only in HBM.

``gen_ses_device`` / ``gen_svm_device`` draw the same DISTRIBUTIONS as
``instances.gen_ses`` / ``gen_svm`` (R/instances.py:155-199) directly on the GPU through
``sc_create_generated``: a counter-based Philox4x32-10 keyed by (seed, global row), so a
row-sharded job generates each rank's rows on that rank and the instance is the same for
every world size.  The bits differ from numpy's PCG64 stream (only the distribution
matches), so these instances have no CPU-reference parity; they exist for the sizes the
host cannot hold (C4: 8 GB, C5: 82 GB).  The SVM separating axis is drawn on the host
exactly as gen_svm draws it (first ``standard_normal(d)`` of ``default_rng(seed)``).

The descriptors are accepted wherever an instance is: ``solve_ses(DeviceSes, eps)`` and
``solve_svm(DeviceSvm, eps)`` run the reference's search over the resident rows.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _native as nat
from .meta import DeviceProblem
from .shard import Comm, ShardedDeviceProblem, _connect, fold_ranks, red_ops, row_ranges

_KV_VEC = 12   # SVM reduced vector: [TP, TQ, M, 9 extremes, GP[d], GQ[d]]


@dataclass
class DeviceSes:
    dev: DeviceProblem
    n: int
    d: int
    D: float
    v1: np.ndarray
    seed: int
    dist: str

    def close(self) -> None:
        self.dev.close()


@dataclass
class DeviceSvm:
    dev: DeviceProblem
    n1: int
    n2: int
    d: int
    D: float
    axis: np.ndarray
    w0: np.ndarray          # P mean - Q mean (seed direction, R/svm.py:194-199)
    seed: int
    gap: float

    def close(self) -> None:
        self.dev.close()


def svm_axis(d: int, seed: int) -> np.ndarray:
    axis = np.random.default_rng(seed).standard_normal(d)
    return axis / np.linalg.norm(axis)


def _svm_seed_direction(red0: np.ndarray, d: int, n1: int, n2: int) -> np.ndarray:
    gp = red0[_KV_VEC:_KV_VEC + d]
    gq = red0[_KV_VEC + d:_KV_VEC + 2 * d]
    return gp / n1 - gq / n2


def gen_ses_device(n: int, d: int, seed: int, dist: str = "gaussian", grid: int = 0,
                   device: int = 0, engine: Optional[nat.Engine] = None,
                   comm: Optional[Comm] = None) -> DeviceSes:
    """SES instance of n points in R^d (zero radii) drawn on the device.  With ``comm``
    (world > 1) this rank draws and keeps only its row range."""
    from .ses import ses_cone
    if n < 2 or d < 1:
        raise ValueError("need n >= 2 and d >= 1")
    if dist not in nat.GEN_DISTS:
        raise ValueError(f"dist must be one of {tuple(nat.GEN_DISTS)}")
    eng = engine if engine is not None else nat.cuda_engine()
    if comm is None or comm.world <= 1:
        h, D, v1 = eng.create_generated(nat.SC_SES, n, d, seed, nat.GEN_DISTS[dist],
                                        grid=grid, device=device)
        return DeviceSes(DeviceProblem(h, ses_cone(n, d), nat.SC_SES), n, d, D, v1, seed, dist)
    r0, r1 = row_ranges(n, comm.world)[comm.rank]
    h, D, v1 = eng.create_generated(nat.SC_SES, n, d, seed, nat.GEN_DISTS[dist], grid=grid,
                                    device=device, shard=(comm.world, comm.rank, r0, r1 - r0))
    D = float(comm.all_gather_array(np.array([D])).max())
    h.set_range(D)
    h.set_globals(fold_ranks(comm.all_gather_array(h.local_red0()), red_ops(nat.SC_SES, d)),
                  v1, 0.0)
    dev = ShardedDeviceProblem(h, ses_cone(n, d), nat.SC_SES, comm)
    _connect(h, comm, nat.SC_SES, d, dev)
    return DeviceSes(dev, n, d, D, v1, seed, dist)


def gen_svm_device(n1: int, n2: int, d: int, seed: int, gap: float = 1.0, grid: int = 0,
                   device: int = 0, engine: Optional[nat.Engine] = None,
                   comm: Optional[Comm] = None) -> DeviceSvm:
    """Two unit-ball clusters shifted by +-(1 + gap/2) along a random axis (the gen_svm
    distribution), drawn on the device; rows P (n1) then Q (n2)."""
    from .svm import svm_cone
    if n1 < 1 or n2 < 1 or d < 1:
        raise ValueError("need n1, n2 >= 1 and d >= 1")
    if gap <= 0:
        raise ValueError("gap must be positive")
    eng = engine if engine is not None else nat.cuda_engine()
    axis = svm_axis(d, seed)
    n = n1 + n2
    if comm is None or comm.world <= 1:
        h, D, _ = eng.create_generated(nat.SC_SVM, n, d, seed, nat.SC_GEN_SVM_CLUSTERS, n1=n1,
                                       gap=gap, direction=axis, grid=grid, device=device)
        w0 = _svm_seed_direction(h.local_red0(), d, n1, n2)
        return DeviceSvm(DeviceProblem(h, svm_cone(n), nat.SC_SVM), n1, n2, d, D, axis, w0,
                         seed, gap)
    r0, r1 = row_ranges(n, comm.world)[comm.rank]
    h, D, _ = eng.create_generated(nat.SC_SVM, n, d, seed, nat.SC_GEN_SVM_CLUSTERS, n1=n1,
                                   gap=gap, direction=axis, grid=grid, device=device,
                                   shard=(comm.world, comm.rank, r0, r1 - r0))
    D = float(comm.all_gather_array(np.array([D])).max())
    h.set_range(D)
    red0 = fold_ranks(comm.all_gather_array(h.local_red0()), red_ops(nat.SC_SVM, d))
    h.set_globals(red0)
    dev = ShardedDeviceProblem(h, svm_cone(n), nat.SC_SVM, comm)
    _connect(h, comm, nat.SC_SVM, d, dev)
    return DeviceSvm(dev, n1, n2, d, D, axis, _svm_seed_direction(red0, d, n1, n2), seed, gap)
