"""Z-order point filter on the GPU (drop-in for morton.py).

``filter_cloud`` runs capt_filter_cloud (csrc/capt_filter.cu): per axis
permutation a bounds reduction, float64 quantisation to the 21-bit lattice,
63-bit key interleave, a stable radix sort by (key, original index), the
greedy gap scan as a parallel next-pointer + pointer-jumping chain walk, and
the orphan repair.  Output is bit-identical to morton.filter_cloud
(morton.py:185-236).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .cloud import PointCloud

__all__ = ["FilterConfig", "axis_bits", "filter_cloud", "reach_filter"]


def axis_bits(k: int) -> int:
    """Quantised bits per axis (morton.py:36-38)."""
    return min(21, 63 // k)


@dataclass(frozen=True)
class FilterConfig:
    """Filter radius plus optional reachability constraint (morton.py:48-67)."""

    r_filter: float
    base: Optional[np.ndarray] = None
    max_reach: Optional[float] = None

    def __post_init__(self):
        if not (np.isfinite(self.r_filter) and self.r_filter >= 0):
            raise ValueError(f"r_filter must be >= 0, got {self.r_filter}")
        if (self.base is None) != (self.max_reach is None):
            raise ValueError("base and max_reach must be given together")
        if self.max_reach is not None and not self.max_reach > 0:
            raise ValueError("max_reach must be > 0")
        if self.base is not None:
            b = np.asarray(self.base, dtype=np.float64)
            if not np.all(np.isfinite(b)):
                raise ValueError("reach base must be finite")
            object.__setattr__(self, "base", b)


def _run_filter(pts: np.ndarray, r_filter: float, base, max_reach, device=None) -> np.ndarray:
    k = pts.shape[1]
    out = np.empty((max(len(pts), 1), k), np.float32)
    n_out = C.c_int64(0)
    has = base is not None
    b = np.ascontiguousarray(base if has else np.zeros(k), dtype=np.float64)
    dev = _lib.default_device() if device is None else int(device)
    rc = _lib.lib().capt_filter_cloud(dev, k, pts.ctypes.data, len(pts), float(r_filter),
                                      int(has), b.ctypes.data, float(max_reach) if has else 0.0,
                                      _lib.HOST_IO, out.ctypes.data, C.byref(n_out), None)
    _lib.check(rc, "capt_filter_cloud")
    return out[: n_out.value].copy()


def reach_filter(cloud: PointCloud, base, max_reach: float, device=None) -> PointCloud:
    """Keep exactly the points within max_reach of base (morton.py:173-182)."""
    if not max_reach > 0:
        raise ValueError("max_reach must be > 0")
    if len(cloud) == 0:
        return cloud
    # reach-only: a filter radius of -1 keeps every survivor of the reach pass
    return PointCloud(_run_filter(cloud.points, -1.0, np.asarray(base, np.float64),
                                  float(max_reach), device))


def filter_cloud(cloud: PointCloud, cfg: FilterConfig, device=None) -> PointCloud:
    """Z-order-curve downsampling, one pass per axis permutation (morton.py:185-236)."""
    if not isinstance(cloud, PointCloud):
        cloud = PointCloud(cloud)
    if len(cloud) == 0:
        return PointCloud(cloud.points)
    return PointCloud(_run_filter(cloud.points, cfg.r_filter, cfg.base, cfg.max_reach, device))
