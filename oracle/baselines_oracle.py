"""CPU restatement of the reference's verification baselines (TEST INFRASTRUCTURE ONLY).

Restates ``symcone.baselines`` (R = /root/reference/pkg/src/symcone/): ``_bc_iterate`` /
``meb_baseline`` (R/baselines.py:34-85) and ``_gilbert_iterate`` / ``gilbert_baseline``
(R/baselines.py:88-161).  The numba loops sum over columns sequentially with separate
multiplies and adds; here the row loop is vectorised with numpy but every column sum keeps
that order (s += diff * diff, column by column), so the values and argmax/argmin choices
are the reference's bit for bit (pinned by tests/golden/baselines.json, generated from the
reference by tests/golden/make_golden.py).  Only tests import this module.
"""
from __future__ import annotations

import math

import numpy as np


def _row_sq_dist(X: np.ndarray, c: np.ndarray) -> np.ndarray:
    s = np.zeros(X.shape[0])
    for j in range(X.shape[1]):
        diff = c[j] - X[:, j]
        s += diff * diff
    return s


def _row_dot(X: np.ndarray, z: np.ndarray) -> np.ndarray:
    s = np.zeros(X.shape[0])
    for k in range(X.shape[1]):
        s += X[:, k] * z[k]
    return s


def bc_iterate(centers: np.ndarray, radii: np.ndarray, iters: int) -> np.ndarray:
    """R/baselines.py:35-62."""
    c = centers[0].copy()
    d = centers.shape[1]
    for t in range(1, iters + 1):
        v = np.sqrt(_row_sq_dist(centers, c)) + radii
        far_i = int(np.argmax(v))            # first index of the max (strict > scan)
        if not v[far_i] > -1.0:
            far_i = 0
        s = 0.0
        for j in range(d):
            diff = centers[far_i, j] - c[j]
            s += diff * diff
        dist = math.sqrt(s)
        step = 1.0 / (t + 1.0)
        if dist > 0.0:
            scale = 1.0 + radii[far_i] / dist
            for j in range(d):
                c[j] += step * scale * (centers[far_i, j] - c[j])
    return c


def meb_baseline(points, radii=None, eps_base: float = 1e-3):
    """R/baselines.py:65-85: (value, centre, iterations)."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    rad = np.zeros(pts.shape[0]) if radii is None else np.ascontiguousarray(radii, np.float64)
    iters = math.ceil(1.0 / eps_base ** 2)
    c = bc_iterate(pts, rad, iters)
    value = float((np.linalg.norm(pts - c, axis=1) + rad).max())
    return value, c, iters


def gilbert_iterate(P: np.ndarray, Q: np.ndarray, gap_tol: float, max_iters: int):
    """R/baselines.py:89-146: (mu, gam, z, gap, it)."""
    n1, d = P.shape
    n2 = Q.shape[0]
    mu = np.zeros(n1)
    gam = np.zeros(n2)
    mu[0] = 1.0
    gam[0] = 1.0
    z = np.empty(d)
    for k in range(d):
        z[k] = P[0, k] - Q[0, k]
    gap = math.inf
    it = 0
    for it in range(1, max_iters + 1):
        sp = _row_dot(P, z)
        best_i = int(np.argmin(sp))          # first index of the min (strict < scan)
        if not sp[best_i] < math.inf:
            best_i = 0
        sq = _row_dot(Q, z)
        best_j = int(np.argmax(sq))
        if not sq[best_j] > -math.inf:
            best_j = 0
        zdiff = 0.0
        denom = 0.0
        for k in range(d):
            dk = (P[best_i, k] - Q[best_j, k]) - z[k]
            zdiff += z[k] * dk
            denom += dk * dk
        gap = -2.0 * zdiff
        if gap < gap_tol:
            break
        if denom == 0.0:
            break
        lam = -zdiff / denom
        if lam > 1.0:
            lam = 1.0
        if lam <= 0.0:
            break
        mu *= 1.0 - lam
        gam *= 1.0 - lam
        mu[best_i] += lam
        gam[best_j] += lam
        for k in range(d):
            z[k] += lam * ((P[best_i, k] - Q[best_j, k]) - z[k])
    return mu, gam, z, gap, it


def gilbert_baseline(P, Q, gap_tol: float = 1e-6, max_iters: int = 10 ** 6):
    """R/baselines.py:149-161: (value, gap, iterations, mu, gam)."""
    P = np.ascontiguousarray(P, dtype=np.float64)
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    mu, gam, z, gap, it = gilbert_iterate(P, Q, gap_tol, max_iters)
    return float(np.linalg.norm(z)), float(gap), int(it), mu, gam
