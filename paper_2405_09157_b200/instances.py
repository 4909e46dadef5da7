"""Instance generators and the text instance format (API of R/instances.py).

The generators issue the same ``numpy.random.default_rng`` call sequence as
the reference (R/instances.py:155-199), so a (n, d, seed, dist) tuple names
the same point set in both code bases (pinned by tests/golden/generators.json).
The text format is the reference's: a header ``ses <n> <d>`` or
``svm <n1> <n2> <d>``, ``#`` comment lines, one row per point, 17 significant
digits.  Binary ``.npz`` instances are added for sizes where text is
impractical (80 GB at C5).
"""
from __future__ import annotations

import io
import os

import numpy as np

from .ses import SesInstance
from .svm import SvmInstance

SES_DISTS = ("uniform-ball", "gaussian", "sphere-surface")


class InstanceFormatError(ValueError):
    pass


def _unit_rows(rng, k: int, d: int) -> np.ndarray:
    g = rng.standard_normal((k, d))
    g /= np.linalg.norm(g, axis=1, keepdims=True)
    return g


def gen_ses(n: int, d: int, seed: int, dist: str = "gaussian") -> SesInstance:
    if n < 2 or d < 1:
        raise ValueError("need n >= 2 and d >= 1")
    if dist not in SES_DISTS:
        raise ValueError(f"dist must be one of {SES_DISTS}")
    rng = np.random.default_rng(seed)
    if dist == "gaussian":
        pts = rng.standard_normal((n, d))
    elif dist == "uniform-ball":
        pts = _unit_rows(rng, n, d) * rng.random(n)[:, None] ** (1.0 / d)
    else:  # antipodal unit pairs pin the optimum to radius 1 about the origin
        half = n // 2
        u = _unit_rows(rng, half + n % 2, d)
        pts = np.concatenate([u[:half], -u[:half], u[half:]])
    return SesInstance(centers=pts, radii=np.zeros(n))


def gen_svm(n1: int, n2: int, d: int, seed: int,
            gap: float = 1.0) -> tuple[SvmInstance, np.ndarray]:
    if n1 < 1 or n2 < 1 or d < 1:
        raise ValueError("need n1, n2 >= 1 and d >= 1")
    if gap <= 0:
        raise ValueError("gap must be positive")
    rng = np.random.default_rng(seed)
    axis = rng.standard_normal(d)
    axis /= np.linalg.norm(axis)
    shift = (1.0 + gap / 2.0) * axis

    def unit_ball(k):
        return _unit_rows(rng, k, d) * rng.random(k)[:, None] ** (1.0 / d)

    P = unit_ball(n1) + shift
    Q = unit_ball(n2) - shift
    return SvmInstance(P=P, Q=Q), axis


def _num(x: float) -> str:
    return format(float(x), ".17g")


def serialize_ses(inst: SesInstance, comments: list[str] | None = None) -> str:
    buf = io.StringIO()
    buf.write(f"ses {inst.n} {inst.d}\n")
    for c in comments or []:
        buf.write(f"# {c}\n")
    for row, r in zip(inst.centers, inst.radii):
        buf.write(" ".join(map(_num, row)) + " " + _num(r) + "\n")
    return buf.getvalue()


def serialize_svm(inst: SvmInstance, comments: list[str] | None = None) -> str:
    buf = io.StringIO()
    buf.write(f"svm {inst.n1} {inst.n2} {inst.d}\n")
    for c in comments or []:
        buf.write(f"# {c}\n")
    for block in (inst.P, inst.Q):
        for row in block:
            buf.write(" ".join(map(_num, row)) + "\n")
    return buf.getvalue()


def _rows(lines: list[str], count: int, width: int) -> np.ndarray:
    if len(lines) != count:
        raise InstanceFormatError(f"expected {count} data rows, found {len(lines)}")
    out = np.empty((count, width))
    for i, ln in enumerate(lines):
        vals = ln.split()
        if len(vals) != width:
            raise InstanceFormatError(f"row {i}: expected {width} values, found {len(vals)}")
        out[i] = [float(v) for v in vals]
    if not np.isfinite(out).all():
        raise InstanceFormatError("non-finite value in instance")
    return out


def parse(text: str) -> SesInstance | SvmInstance:
    body = [ln.strip() for ln in text.splitlines()]
    body = [ln for ln in body if ln and not ln.startswith("#")]
    if not body:
        raise InstanceFormatError("empty instance file")
    head = body[0].split()
    try:
        if head[0] == "ses":
            if len(head) != 3:
                raise InstanceFormatError(f"bad ses header: {body[0]!r}")
            n, d = int(head[1]), int(head[2])
            rows = _rows(body[1:], n, d + 1)
            return SesInstance(centers=rows[:, :d], radii=rows[:, d])
        if head[0] == "svm":
            if len(head) != 4:
                raise InstanceFormatError(f"bad svm header: {body[0]!r}")
            n1, n2, d = int(head[1]), int(head[2]), int(head[3])
            rows = _rows(body[1:], n1 + n2, d)
            return SvmInstance(P=rows[:n1], Q=rows[n1:])
    except InstanceFormatError:
        raise
    except (ValueError, IndexError) as exc:
        raise InstanceFormatError(str(exc)) from exc
    raise InstanceFormatError(f"unknown problem kind {head[0]!r}")


def _is_npy_dir(path: str) -> bool:
    return path.endswith(".npyd") or (os.path.isdir(path) and (
        os.path.exists(os.path.join(path, "centers.npy")) or
        os.path.exists(os.path.join(path, "P.npy"))))


def load(path: str, mmap: bool = True) -> SesInstance | SvmInstance:
    """Text (the reference's format, R/instances.py:1-9), ``.npz``, or a binary instance
    directory (``*.npyd``: centers.npy + radii.npy, or P.npy + Q.npy).  Directories are
    memory-mapped by default: an instance larger than host RAM streams from the page
    cache through the engine's pinned staging buffers at upload."""
    if _is_npy_dir(path):
        mode = "r" if mmap else None
        if os.path.exists(os.path.join(path, "centers.npy")):
            return SesInstance(centers=np.load(os.path.join(path, "centers.npy"), mmap_mode=mode),
                               radii=np.load(os.path.join(path, "radii.npy"), mmap_mode=mode))
        return SvmInstance(P=np.load(os.path.join(path, "P.npy"), mmap_mode=mode),
                           Q=np.load(os.path.join(path, "Q.npy"), mmap_mode=mode))
    if path.endswith(".npz"):
        z = np.load(path)
        if "centers" in z:
            return SesInstance(centers=z["centers"], radii=z["radii"])
        return SvmInstance(P=z["P"], Q=z["Q"])
    with open(path, "r", encoding="utf-8") as fh:
        return parse(fh.read())


def save(path: str, inst_or_text) -> None:
    if path.endswith(".npyd"):
        os.makedirs(path, exist_ok=True)
        if isinstance(inst_or_text, SesInstance):
            np.save(os.path.join(path, "centers.npy"), inst_or_text.centers)
            np.save(os.path.join(path, "radii.npy"), inst_or_text.radii)
        else:
            np.save(os.path.join(path, "P.npy"), inst_or_text.P)
            np.save(os.path.join(path, "Q.npy"), inst_or_text.Q)
        return
    if path.endswith(".npz"):
        if isinstance(inst_or_text, SesInstance):
            np.savez(path, centers=inst_or_text.centers, radii=inst_or_text.radii)
        else:
            np.savez(path, P=inst_or_text.P, Q=inst_or_text.Q)
        return
    text = inst_or_text if isinstance(inst_or_text, str) else (
        serialize_ses(inst_or_text) if isinstance(inst_or_text, SesInstance)
        else serialize_svm(inst_or_text))
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write(text)
