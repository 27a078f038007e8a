"""Collision queries against a device tree (drop-in for query.py).

Every entry point runs the sm_100a kernels of libcapt_b200 through
``capt_query`` (include/capt_b200.h); there is no host fallback.  Host numpy
inputs take the CAPT_HOST_IO path (copy in, kernel, copy the bit mask out);
CUDA tensors stay on the device.  Verdicts are bit-identical to the
reference's float64 evaluation (see csrc/capt_query.cu).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .geom import Sphere
from .tree import Capt, leaf_index, leaf_indices  # noqa: F401  (re-export like query.py)

__all__ = ["SphereBatch", "QueryOutcome", "collides", "collides_unchecked",
           "collides_batch", "collides_any", "collides_many", "query_bits",
           "DEFAULT_LANE_WIDTH"]

DEFAULT_LANE_WIDTH = 8
N_COUNTERS = 6


def _check_radius(tree: Capt, r: float) -> None:
    """query.py:30-34 -- same message."""
    if not (tree.r_min <= r <= tree.r_max):
        raise ValueError(
            f"radius {r} outside the tree's exactness band "
            f"[{tree.r_min}, {tree.r_max}]")


@dataclass
class SphereBatch:
    """Fixed-width group of spheres with a per-lane validity mask (query.py:37-78)."""

    centers: np.ndarray
    radii: np.ndarray
    mask: np.ndarray

    def __post_init__(self):
        self.centers = np.asarray(self.centers, dtype=np.float64)
        self.radii = np.asarray(self.radii, dtype=np.float64)
        self.mask = np.asarray(self.mask, dtype=bool)
        L = self.centers.shape[0]
        if L == 0 or L & (L - 1):
            raise ValueError(f"lane width {L} is not a power of two")
        if self.radii.shape != (L,) or self.mask.shape != (L,):
            raise ValueError("centers, radii, and mask lengths disagree")

    @property
    def width(self) -> int:
        return self.centers.shape[0]

    @classmethod
    def from_spheres(cls, spheres: Sequence[Sphere],
                     lane_width: int = DEFAULT_LANE_WIDTH) -> "SphereBatch":
        if not spheres or len(spheres) > lane_width:
            raise ValueError("need 1..lane_width spheres")
        first = spheres[0]
        centers = np.tile(first.center, (lane_width, 1))
        radii = np.full(lane_width, first.radius, dtype=np.float64)
        mask = np.zeros(lane_width, dtype=bool)
        for i, s in enumerate(spheres):
            centers[i] = s.center
            radii[i] = s.radius
            mask[i] = True
        return cls(centers, radii, mask)


@dataclass
class QueryOutcome:
    """Result of a batched query (query.py:81-93)."""

    any_collision: bool
    lane_bits: Optional[np.ndarray] = None
    aabb_rejections: Optional[int] = None
    points_scanned: Optional[int] = None


# ---------------------------------------------------------------------------
# low-level calls
# ---------------------------------------------------------------------------

def _host_inputs(tree: Capt, centers, radii):
    """Contiguous host arrays for a CAPT_HOST_IO call: fp32 pairs as they
    are; anything else as float64 (the reference converts with
    np.asarray(float64), query.py:192-193).  Float64 batches go to the
    device unchanged: capt_query sends every sphere whose values are fp32
    values through the fp32 kernels (bit-identical) and the rest through
    the float64 path, on the device."""
    c = np.asarray(centers)
    r = np.asarray(radii)
    if c.dtype == np.float32 and r.dtype == np.float32:
        c = np.ascontiguousarray(c)
        r = np.ascontiguousarray(r)
        f64 = 0
    else:
        c = np.ascontiguousarray(c, dtype=np.float64)
        r = np.ascontiguousarray(r, dtype=np.float64)
        f64 = _lib.INPUT_F64
    c = c.reshape(-1, tree.k)
    r = r.reshape(-1)
    if len(c) != len(r):
        raise ValueError("centers and radii lengths disagree")
    return c, r, f64


def _host_query(tree: Capt, c, r, f64: int, lane_width: int = 1, lane_mask=None,
                prefilter: bool = True, check: bool = True, stats: bool = False,
                mode: int = 0):
    """CAPT_HOST_IO call.  Returns (verdicts bool array, counters or None,
    first_bad)."""
    n = len(r)
    ng = n // lane_width
    words = np.zeros(max((ng + 31) // 32, 1), np.uint32)
    cnt = np.zeros(N_COUNTERS, np.uint64)
    bad = C.c_int64(-1)
    m = None
    if lane_mask is not None:
        m = np.ascontiguousarray(lane_mask, dtype=np.uint8).reshape(-1)
    flags = _lib.HOST_IO | f64 | mode
    if prefilter:
        flags |= _lib.PREFILTER
    if check:
        flags |= _lib.CHECK_RADII
    if stats:
        flags |= _lib.STATS
    rc = _lib.lib().capt_query(tree.handle, c.ctypes.data, r.ctypes.data, n, int(lane_width),
                               None if m is None else m.ctypes.data, flags, words.ctypes.data,
                               cnt.ctypes.data, C.byref(bad), None)
    if rc == _lib.CAPT_ERANGE:
        return None, None, int(bad.value)
    _lib.check(rc, "capt_query")
    bits = np.unpackbits(words.view(np.uint8), bitorder="little")[:ng].view(bool)
    return bits, (cnt if stats else None), int(bad.value)


def query_bits(tree: Capt, centers, radii, lane_width: int = 1, lane_mask=None,
               out=None, counters=None, first_bad=None, use_aabb_prefilter: bool = True,
               check_radii: bool = True, mode: int = 0, stream=None):
    """Device-resident query: CUDA tensors in, packed uint32 verdict words out
    (bit g % 32 of word g // 32).  Asynchronous on ``stream`` (default: the
    current torch stream); nothing is copied to the host."""
    import torch
    c = centers if centers.is_contiguous() else centers.contiguous()
    r = radii if radii.is_contiguous() else radii.contiguous()
    flags = mode
    if c.dtype == torch.float64 or r.dtype == torch.float64:
        c, r = c.to(torch.float64), r.to(torch.float64)
        flags |= _lib.INPUT_F64
    n = int(r.numel())
    ng = n // lane_width
    nw = max((ng + 31) // 32, 1)
    if out is None:
        out = torch.empty(nw, dtype=torch.int32, device=c.device)
    if use_aabb_prefilter:
        flags |= _lib.PREFILTER
    if check_radii and first_bad is not None:
        flags |= _lib.CHECK_RADII
    if counters is not None:
        flags |= _lib.STATS
    if stream is None:
        stream = torch.cuda.current_stream(c.device).cuda_stream
    rc = _lib.lib().capt_query(tree.handle, c.data_ptr(), r.data_ptr(), n, int(lane_width),
                               _lib.ptr(lane_mask), flags, out.data_ptr(), _lib.ptr(counters),
                               _lib.ptr(first_bad), stream)
    _lib.check(rc, "capt_query")
    return out


def _unpack_device(words, n):
    import torch
    shifts = torch.arange(32, device=words.device, dtype=torch.int32)
    bits = (words.view(torch.int32)[:, None] >> shifts[None, :]) & 1
    return bits.reshape(-1)[:n].to(torch.bool)


# ---------------------------------------------------------------------------
# reference API
# ---------------------------------------------------------------------------

def collides_many(tree: Capt, centers, radii, use_aabb_prefilter: bool = True,
                  check_radii: bool = True):
    """Bulk verdicts (query.py:184-219): verdict[i] == collides(tree, Sphere(c_i, r_i)).

    numpy in -> numpy bool out; CUDA tensors in -> CUDA bool tensor out."""
    if hasattr(centers, "data_ptr") and getattr(centers, "is_cuda", False):
        import torch
        n = int(radii.numel())
        bad = torch.full((1,), -1, dtype=torch.int64, device=centers.device) if check_radii else None
        words = query_bits(tree, centers, radii, 1, first_bad=bad,
                           use_aabb_prefilter=use_aabb_prefilter, check_radii=check_radii)
        if check_radii:
            b = int(bad.item())
            if b >= 0:
                _check_radius(tree, float(radii[b].item()))
        return _unpack_device(words, n)
    c, r, f64 = _host_inputs(tree, centers, radii)
    if len(r) == 0:
        return np.zeros(0, dtype=bool)
    bits, _, bad = _host_query(tree, c, r, f64, 1, None, use_aabb_prefilter, check_radii)
    if bits is None:
        _check_radius(tree, float(r[bad]))
    return bits


def collides_unchecked(tree: Capt, s: Sphere, use_aabb_prefilter: bool = True) -> bool:
    """Scalar check without the radius-band guard (query.py:102-114)."""
    c = np.asarray(s.center, np.float64).reshape(1, tree.k)
    r = np.array([s.radius], np.float64)
    bits, _, _ = _host_query(tree, c, r, _lib.INPUT_F64, 1, None, use_aabb_prefilter, False)
    return bool(bits[0])


def collides(tree: Capt, s: Sphere, use_aabb_prefilter: bool = True) -> bool:
    """True iff some cloud point lies within s.radius of s.center (query.py:117-123)."""
    _check_radius(tree, s.radius)
    return collides_unchecked(tree, s, use_aabb_prefilter=use_aabb_prefilter)


def collides_batch(tree: Capt, batch: SphereBatch, use_aabb_prefilter: bool = True,
                   want_lane_bits: bool = False, collect_stats: bool = False) -> QueryOutcome:
    """Lockstep lanes with validity mask and early exit (query.py:126-167)."""
    for r in batch.radii[batch.mask]:
        _check_radius(tree, float(r))
    L = batch.width
    c, r = batch.centers, batch.radii
    mask = batch.mask.astype(np.uint8)
    f64 = _lib.INPUT_F64
    if want_lane_bits:
        bits, cnt, _ = _host_query(tree, c, r, f64, 1, mask, use_aabb_prefilter, False,
                                   collect_stats)
        return QueryOutcome(
            any_collision=bool(bits.any()), lane_bits=bits,
            aabb_rejections=int(cnt[4]) if collect_stats else None,
            points_scanned=int(cnt[2]) if collect_stats else None)
    if L <= 32:
        bits, cnt, _ = _host_query(tree, c, r, f64, L, mask, use_aabb_prefilter, False,
                                   collect_stats)
        return QueryOutcome(
            any_collision=bool(bits[0]),
            aabb_rejections=int(cnt[4]) if collect_stats else None,
            points_scanned=int(cnt[2]) if collect_stats else None)
    # wider than a warp: 32-lane sub-groups, scanned in order with early exit
    bits, cnt, _ = _host_query(tree, c, r, f64, 32, mask, use_aabb_prefilter, False,
                               collect_stats)
    any_hit = bool(bits.any())
    if not collect_stats:
        return QueryOutcome(any_collision=any_hit)
    scanned = 0
    for g in range(L // 32):
        s = slice(32 * g, 32 * (g + 1))
        b, cg, _ = _host_query(tree, c[s], r[s], f64, 32, mask[s], use_aabb_prefilter,
                               False, True)
        scanned += int(cg[2])
        if b[0]:
            break
    return QueryOutcome(any_collision=any_hit, aabb_rejections=int(cnt[4]),
                        points_scanned=scanned)


def collides_any(tree: Capt, spheres: Sequence[Sphere], lane_width: int = DEFAULT_LANE_WIDTH,
                 use_aabb_prefilter: bool = True) -> bool:
    """OR over a sphere list in lane_width chunks with early termination
    (query.py:170-181): a chunk's radius check runs only if no earlier chunk
    collided, so a bad radius raises iff its chunk is not after the first
    colliding chunk."""
    if not spheres:
        return False
    if lane_width < 1 or lane_width & (lane_width - 1):
        raise ValueError(f"lane width {lane_width} is not a power of two")
    n = len(spheres)
    ng = (n + lane_width - 1) // lane_width
    c = np.empty((ng * lane_width, tree.k), np.float64)
    r = np.empty(ng * lane_width, np.float64)
    m = np.zeros(ng * lane_width, np.uint8)
    for i, s in enumerate(spheres):
        c[i] = s.center
        r[i] = s.radius
        m[i] = 1
    c[n:] = spheres[(n - 1) // lane_width * lane_width].center
    r[n:] = spheres[(n - 1) // lane_width * lane_width].radius
    L = min(lane_width, 32)
    bits, _, _ = _host_query(tree, c, r, _lib.INPUT_F64, L, m, use_aabb_prefilter, False)
    if lane_width > 32:
        bits = bits.reshape(ng, lane_width // 32).any(1)
    hit_chunks = np.nonzero(bits)[0]
    first_hit = int(hit_chunks[0]) if len(hit_chunks) else ng
    bad = np.nonzero(~((r >= tree.r_min) & (r <= tree.r_max)) & (m != 0))[0]
    if len(bad) and bad[0] // lane_width <= first_hit:
        _check_radius(tree, float(r[bad[0]]))
    return first_hit < ng
