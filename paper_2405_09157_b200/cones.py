"""Cone shape descriptors used at the API boundary (R/cones.py:33-116).

Only the shape information travels: which blocks, the ambient dimension and
the rank (which enters ln r and the iteration bound).  The algebra itself
(spectral exponential, norms) runs on the device inside the fused pass.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from functools import cached_property

import numpy as np

SQRT2 = math.sqrt(2.0)


@dataclass(frozen=True)
class Orthant:
    """Nonnegative-orthant block, rank == dim."""
    dim: int


@dataclass(frozen=True)
class SecondOrder:
    """Second-order-cone block with a vector part of dimension ``dim``
    (dim + 1 coordinates, vector part first, rank 2)."""
    dim: int


@dataclass(frozen=True)
class Cone:
    """Ordered product of blocks.  Large uniform products are described by a
    single (block, count) pair so an n = 10^7 cone costs O(1) to describe."""

    block: Orthant | SecondOrder
    count: int = 1

    def __post_init__(self):
        if not isinstance(self.block, (Orthant, SecondOrder)):
            raise TypeError(f"unsupported block type: {self.block!r}")
        if self.block.dim < 1 or self.count < 1:
            raise ValueError("block dimension and count must be >= 1")

    @cached_property
    def ambient_dim(self) -> int:
        b = self.block
        return self.count * (b.dim if isinstance(b, Orthant) else b.dim + 1)

    @cached_property
    def rank(self) -> int:
        b = self.block
        return self.count * (b.dim if isinstance(b, Orthant) else 2)

    @property
    def blocks(self) -> tuple:
        return (self.block,) * self.count


@dataclass(frozen=True, eq=False)
class Element:
    """A point of the algebra (materialised only on request, e.g. p_last)."""

    cone: Cone
    coords: np.ndarray

    def __post_init__(self):
        c = np.asarray(self.coords, dtype=np.float64)
        if c.shape != (self.cone.ambient_dim,):
            raise ValueError(f"coords length {c.shape} != ambient dim "
                             f"({self.cone.ambient_dim},)")
        object.__setattr__(self, "coords", c)
