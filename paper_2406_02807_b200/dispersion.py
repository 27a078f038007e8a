"""Cloud dispersion proxy on the device.

``dispersion_stats`` mirrors oracle.py:141-158: the distance from every point
to its nearest other point (a float64 k-d tree query with k=2 in the
reference; an exact float64 brute force on the GPU here, capt_nn_distances),
summarised with numpy's mean / median / 95th percentile exactly as the
reference does.  ``safe_filter_radius`` is the advisory Lemma-2 helper of
morton.py:239-245.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .cloud import PointCloud

__all__ = ["DispersionStats", "dispersion_stats", "nn_distances", "safe_filter_radius"]


@dataclass
class DispersionStats:
    mean: float
    median: float
    p95: float
    count: int


def nn_distances(cloud, device=None) -> np.ndarray:
    """(n,) float64 nearest-other-point distance of every point."""
    pts = cloud.points if isinstance(cloud, PointCloud) else np.asarray(cloud)
    pts = np.ascontiguousarray(pts, dtype=np.float32)
    n = len(pts)
    if n < 2:
        raise ValueError("dispersion needs at least 2 points")
    k = pts.shape[1] if pts.ndim == 2 else 1
    out = np.empty(n, np.float64)
    dev = _lib.default_device() if device is None else int(device)
    _lib.check(_lib.lib().capt_nn_distances(dev, k, pts.ctypes.data, n, _lib.HOST_IO,
                                            out.ctypes.data, None), "capt_nn_distances")
    return out


def dispersion_stats(cloud, device=None) -> DispersionStats:
    """Nearest-neighbour proxy for cloud dispersion (oracle.py:141-158);
    duplicates count as neighbours at distance zero."""
    if len(cloud) < 2:
        raise ValueError("dispersion needs at least 2 points")
    nn = nn_distances(cloud, device)
    return DispersionStats(mean=float(nn.mean()), median=float(np.median(nn)),
                           p95=float(np.percentile(nn, 95)), count=len(nn))


def safe_filter_radius(r_min: float, dispersion: float) -> float:
    """Advisory filter radius r_min - dispersion, never negative
    (morton.py:239-245); not enforced by filter_cloud."""
    return max(0.0, float(r_min) - float(dispersion))
