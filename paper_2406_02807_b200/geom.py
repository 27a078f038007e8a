"""Value types of the reference API (geom.py:49-104): Aabb and Sphere.

Host-side containers only; all distance math runs in the CUDA kernels.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["Aabb", "Sphere"]


@dataclass(frozen=True)
class Aabb:
    """Axis-aligned box (geom.py:49-86); lo = hi = +inf is a padding leaf's box."""

    lo: np.ndarray
    hi: np.ndarray

    def __post_init__(self):
        lo = np.asarray(self.lo, dtype=np.float64)
        hi = np.asarray(self.hi, dtype=np.float64)
        if lo.shape != hi.shape or lo.ndim != 1:
            raise ValueError("lo/hi must be 1-D arrays of equal length")
        if np.any(np.isnan(lo)) or np.any(np.isnan(hi)):
            raise ValueError("box bounds contain NaN")
        if not np.all(lo <= hi):
            raise ValueError("box has lo > hi on some axis")
        object.__setattr__(self, "lo", lo)
        object.__setattr__(self, "hi", hi)

    @property
    def k(self) -> int:
        return self.lo.shape[0]

    def contains(self, p) -> bool:
        p = np.asarray(p, dtype=np.float64)
        return bool(np.all(self.lo <= p) and np.all(p <= self.hi))


@dataclass(frozen=True)
class Sphere:
    """Query primitive (geom.py:89-104): finite centre, finite radius > 0."""

    center: np.ndarray
    radius: float

    def __post_init__(self):
        c = np.asarray(self.center, dtype=np.float64)
        if c.ndim != 1 or not np.all(np.isfinite(c)):
            raise ValueError("sphere center must be a finite 1-D point")
        r = float(self.radius)
        if not (np.isfinite(r) and r > 0):
            raise ValueError(f"sphere radius must be finite and > 0, got {r}")
        object.__setattr__(self, "center", c)
        object.__setattr__(self, "radius", r)
