"""Independent verification solvers on the GPU.

Same API and algorithms as the reference's ``symcone.baselines`` (R/baselines.py): the
Badoiu-Clarkson walk for the minimum enclosing ball of spheres (``meb_baseline``,
R/baselines.py:34-85) and Gilbert / Frank-Wolfe with exact line search for the polytope
distance (``gilbert_baseline``, R/baselines.py:88-161).  They share no code with the SCMWU
engine except the resident instance, so agreement between the two is evidence.  The
reference guards them to n <= 1e5 (R/bench.py:26) because each iteration is a full pass
over the points; here each iteration is one streaming argmax pass of a persistent kernel
(``sc_meb_baseline`` / ``sc_gilbert_baseline``), so they run at the BASELINE sizes.

Inputs are host arrays (uploaded here) or device-resident instances (``DeviceSes`` /
``DeviceSvm`` from devgen, or a ``DeviceProblem``).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native as nat


@dataclass
class BaselineResult:
    value: float
    certificate: object
    iterations: int
    gap: float | None = None


def _ses_handle(points, radii, engine):
    from .devgen import DeviceSes
    from .meta import DeviceProblem
    from .ses import SesInstance, ses_device
    if isinstance(points, DeviceSes):
        return points.dev.handle, None
    if isinstance(points, DeviceProblem):
        return points.handle, None
    pts = np.ascontiguousarray(points, dtype=np.float64)
    if pts.ndim != 2:
        raise ValueError("points must be (n, d)")
    rad = np.zeros(pts.shape[0]) if radii is None else np.ascontiguousarray(radii, np.float64)
    dev = ses_device(SesInstance(centers=pts, radii=rad), D=1.0, engine=engine)
    return dev.handle, dev


def meb_baseline(points, radii=None, eps_base: float = 1e-3,
                 engine: nat.Engine | None = None) -> BaselineResult:
    """Core-set walk toward the far side of the farthest sphere, step 1/(t+1), for
    ceil(1/eps_base^2) steps; the certified covering radius at the final centre is a
    (1 + eps_base)-approximation (R/baselines.py:65-85)."""
    if not 0.0 < eps_base <= 0.1:
        raise ValueError("eps_base must be in (0, 0.1]")
    h, own = _ses_handle(points, radii, engine)
    try:
        if h.prob.n_local == 1:
            raise ValueError("need at least two points")
        iters = math.ceil(1.0 / eps_base ** 2)
        c, value = h.meb_baseline(iters)
        return BaselineResult(value=value, certificate=c, iterations=iters)
    finally:
        if own is not None:
            own.close()


def gilbert_baseline(P, Q=None, gap_tol: float = 1e-6, max_iters: int = 10 ** 6,
                     engine: nat.Engine | None = None) -> BaselineResult:
    """Frank-Wolfe on min |P^T mu - Q^T gam|^2 over the product of simplices with exact
    line search; stops when the linearisation gap drops below gap_tol (R/baselines.py:
    149-161).  ``P`` may be a DeviceSvm / DeviceProblem (then ``Q`` is unused)."""
    if gap_tol <= 0:
        raise ValueError("gap_tol must be positive")
    from .devgen import DeviceSvm
    from .meta import DeviceProblem
    from .svm import SvmInstance, svm_device
    own = None
    if isinstance(P, DeviceSvm):
        h = P.dev.handle
    elif isinstance(P, DeviceProblem):
        h = P.handle
    else:
        inst = SvmInstance(P=np.ascontiguousarray(P, np.float64),
                           Q=np.ascontiguousarray(Q, np.float64))
        own = svm_device(inst, engine=engine)
        h = own.handle
    try:
        value, gap, it, mu, gam = h.gilbert_baseline(gap_tol, max_iters)
        return BaselineResult(value=value, certificate=(mu, gam), iterations=it, gap=gap)
    finally:
        if own is not None:
            own.close()
