"""Device-resident collision-affording point tree (drop-in for tree.py).

``construct`` builds the tree on the GPU (capt_tree_build); ``Capt`` owns a
device slab (include/capt_b200.h) and exposes the reference's arrays
(``tests``, ``aff_lo``, ``aff_hi``, ``offsets``, ``aff_values``) as host copies
exported on first access, so code written against ``captree.Capt``
(tree.py:67-128) keeps working.
"""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from .cloud import PointCloud
from .geom import Aabb

__all__ = ["BuildParams", "BuildStats", "Capt", "construct", "leaf_index",
           "leaf_index_counted", "leaf_indices", "save_capt", "load_capt"]

MAGIC = b"CAPT0001"
_HEADER = struct.Struct("<8sIQQff")


@dataclass(frozen=True)
class BuildParams:
    """Query radius band the tree is built for (tree.py:41-52)."""

    r_min: float
    r_max: float

    def __post_init__(self):
        if not (np.isfinite(self.r_min) and np.isfinite(self.r_max)):
            raise ValueError("r_min and r_max must be finite")
        if not (0 < self.r_min <= self.r_max):
            raise ValueError(f"need 0 < r_min <= r_max, got ({self.r_min}, {self.r_max})")


@dataclass(frozen=True)
class BuildStats:
    """Size and memory summary of a built tree (tree.py:55-64)."""

    n_leaves: int
    n_points: int
    max_affordance: int
    mean_affordance: float
    total_stored: int
    memory_bytes: int


def _as_host(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


class Capt:
    """Immutable tree on one CUDA device.  Safe for concurrent readers.

    ``Capt(k, n_points, r_min, r_max, tests, aff_lo, aff_hi, offsets,
    aff_values)`` uploads a tree given in the reference layout (tree.py:74-97).
    """

    def __init__(self, k: int, n_points: int, r_min: float, r_max: float, tests, aff_lo,
                 aff_hi, offsets, aff_values, device: int | None = None):
        n = len(tests) + 1
        if n & (n - 1):
            raise ValueError(f"leaf count {n} is not a power of two")
        aff_lo = _as_host(aff_lo, np.float32).reshape(-1, k) if np.size(aff_lo) else np.zeros((0, k), np.float32)
        aff_hi = _as_host(aff_hi, np.float32).reshape(-1, k) if np.size(aff_hi) else np.zeros((0, k), np.float32)
        offsets = _as_host(offsets, np.int64)
        if aff_lo.shape != (n, k) or aff_hi.shape != (n, k):
            raise ValueError("affordance box arrays have wrong shape")
        if offsets.shape != (n + 1,):
            raise ValueError("offsets array has wrong shape")
        tests = _as_host(tests, np.float32)
        vals = _as_host(aff_values, np.float32)
        dev = _lib.default_device() if device is None else int(device)
        h = C.c_void_p()
        rc = _lib.lib().capt_tree_create(dev, int(k), n, int(n_points), float(r_min), float(r_max),
                                         tests.ctypes.data if n > 1 else None,
                                         aff_lo.ctypes.data, aff_hi.ctypes.data,
                                         offsets.ctypes.data, vals.ctypes.data, C.byref(h))
        _lib.check(rc, "capt_tree_create")
        self._init_from_handle(h, r_min, r_max)

    # -- construction helpers -------------------------------------------------
    @classmethod
    def _from_handle(cls, handle: C.c_void_p, r_min: float, r_max: float) -> "Capt":
        obj = cls.__new__(cls)
        obj._init_from_handle(handle, r_min, r_max)
        return obj

    def _init_from_handle(self, handle, r_min, r_max):
        self._h = handle
        info = _lib.CaptTreeInfo()
        _lib.check(_lib.lib().capt_tree_info_get(handle, C.byref(info)), "capt_tree_info_get")
        self._info = info
        self.k = int(info.k)
        self.n = int(info.n_leaves)
        self.n_points = int(info.n_points)
        self.r_min = float(r_min)
        self.r_max = float(r_max)
        self.depth = int(info.depth)
        self.device = int(info.device)
        self.n_ties = int(info.n_ties)
        self._host = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.lib().capt_tree_destroy(h)
            except Exception:  # noqa: BLE001 - interpreter shutdown
                pass
            self._h = None
        self._slab_owner = None  # an adopted slab outlives the handle

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    # -- reference-layout views (exported lazily) -----------------------------
    def _export(self):
        if self._host is None:
            n, k = self.n, self.k
            tot = int(self._info.total_stored)
            tests = np.empty(max(n - 1, 1), np.float32)
            lo = np.empty((n, k), np.float32)
            hi = np.empty((n, k), np.float32)
            off = np.empty(n + 1, np.int64)
            vals = np.empty(max(tot * k, 1), np.float32)
            _lib.check(_lib.lib().capt_tree_export(self._h, tests.ctypes.data, lo.ctypes.data,
                                                   hi.ctypes.data, off.ctypes.data,
                                                   vals.ctypes.data), "capt_tree_export")
            self._host = dict(tests=tests[: n - 1], aff_lo=lo, aff_hi=hi, offsets=off,
                              aff_values=vals[: tot * k])
            for a in self._host.values():
                a.setflags(write=False)
        return self._host

    @property
    def tests(self) -> np.ndarray:
        return self._export()["tests"]

    @property
    def aff_lo(self) -> np.ndarray:
        return self._export()["aff_lo"]

    @property
    def aff_hi(self) -> np.ndarray:
        return self._export()["aff_hi"]

    @property
    def offsets(self) -> np.ndarray:
        return self._export()["offsets"]

    @property
    def aff_values(self) -> np.ndarray:
        return self._export()["aff_values"]

    def affordance_set(self, j: int) -> np.ndarray:
        """(m, k) fp32 view of leaf j's set; row 0 is the representative."""
        off = self.offsets
        a, b = off[j], off[j + 1]
        return self.aff_values[a * self.k: b * self.k].reshape(self.k, b - a).T

    def affordance_size(self, j: int) -> int:
        off = self.offsets
        return int(off[j + 1] - off[j])

    def affordance_box(self, j: int) -> Aabb:
        return Aabb(self.aff_lo[j].astype(np.float64), self.aff_hi[j].astype(np.float64))

    def representative(self, j: int) -> np.ndarray:
        return self.affordance_set(j)[0]

    def stats(self) -> BuildStats:
        info = self._info
        n, k = self.n, self.k
        mem = 4 * (n - 1) + 2 * 4 * n * k + 8 * (n + 1) + 4 * int(info.total_stored) * k
        return BuildStats(n_leaves=n, n_points=self.n_points,
                          max_affordance=int(info.max_affordance),
                          mean_affordance=float(info.total_stored) / n,
                          total_stored=int(info.total_stored), memory_bytes=int(mem))

    @property
    def device_bytes(self) -> int:
        return int(self._info.device_bytes)

    def clearance_field(self, cells: bool = False, candidates: bool = False):
        """The tree's clearance field (include/capt_b200.h capt_tree_field):
        a dict of its geometry, plus with ``cells`` the (nz, ny, nx, 8)
        float32 records {witness xyz, nn, kd, candidate count, kd2, k2} (kd2:
        the second record's bound after the witness and k2 more points) and with
        ``candidates`` the (nz, ny, nx, n_cand, 3) candidate offsets
        (p - x0) / q_step (+inf for unused slots); None for trees without
        one (k < 3)."""
        info = _lib.CaptFieldInfo()
        L = _lib.lib()
        if L.capt_tree_field(self._h, C.byref(info), None, None) != _lib.CAPT_OK:
            return None
        out = dict(shape=(info.nz, info.ny, info.nx), n_cells=int(info.n_cells),
                   lo=np.array(info.lo[:], np.float32), h=np.float32(info.h),
                   c0=np.array(info.c0[:], np.float32),
                   box_lo=np.array(info.box_lo[:], np.float32),
                   box_hi=np.array(info.box_hi[:], np.float32), rcap=np.float32(info.rcap),
                   n_cand=int(info.n_cand), q_step=np.float32(info.q_step),
                   q_err=np.float32(info.q_err))
        if cells or candidates:
            buf = np.empty((info.nz, info.ny, info.nx, 8), np.float32) if cells else None
            cb = (np.empty((info.nz, info.ny, info.nx, info.n_cand, 3), np.float32)
                  if candidates else None)
            _lib.check(L.capt_tree_field(self._h, C.byref(info),
                                         None if buf is None else buf.ctypes.data,
                                         None if cb is None else cb.ctypes.data),
                       "capt_tree_field")
            if cells:
                out["cells"] = buf
            if candidates:
                out["candidates"] = cb
        return out

    def field_blocks(self):
        """The clearance field's block table (include/capt_b200.h
        capt_tree_field_blocks): dict(table=(bz, by, bx) uint8, shift, step),
        or None for trees without a field."""
        dims = (C.c_int32 * 4)()
        step = C.c_float(0.0)
        L = _lib.lib()
        if L.capt_tree_field_blocks(self._h, dims, C.byref(step), None) != _lib.CAPT_OK:
            return None
        tab = np.empty((dims[2], dims[1], dims[0]), np.uint8)
        _lib.check(L.capt_tree_field_blocks(self._h, dims, C.byref(step), tab.ctypes.data),
                   "capt_tree_field_blocks")
        return dict(table=tab, shift=int(dims[3]), step=np.float32(step.value))

    # -- replication (multi-GPU) ---------------------------------------------
    def slab_tensor(self):
        """Zero-copy torch uint8 view of the position-independent device slab
        (include/capt_b200.h capt_tree_slab) -- what NCCL broadcasts."""
        import torch
        p, b = C.c_void_p(), C.c_int64()
        _lib.check(_lib.lib().capt_tree_slab(self._h, C.byref(p), C.byref(b)), "capt_tree_slab")

        class _View:
            __cuda_array_interface__ = {"shape": (int(b.value),), "typestr": "|u1",
                                        "data": (int(p.value), False), "version": 3}

        t = torch.as_tensor(_View(), device=torch.device("cuda", self.device))
        t._capt_owner = self  # keep the tree alive while the view exists
        return t

    @classmethod
    def from_slab(cls, slab, device: int | None = None, stream=None,
                  adopt: bool = False) -> "Capt":
        """A tree over a slab (CUDA uint8 tensor) on ``device``: a copy, or with
        ``adopt`` the tensor itself (kept alive by the tree; no second copy of
        a broadcast replica)."""
        dev = slab.device.index if device is None else int(device)
        if adopt and slab.device.index != dev:
            raise ValueError("an adopted slab must live on the tree's device")
        h = C.c_void_p()
        flags = _lib.SLAB_BORROW if adopt else 0
        _lib.check(_lib.lib().capt_tree_from_slab(dev, slab.data_ptr(), int(slab.numel()), flags,
                                                  None if stream is None else int(stream),
                                                  C.byref(h)), "capt_tree_from_slab")
        info = _lib.CaptTreeInfo()
        _lib.check(_lib.lib().capt_tree_info_get(h, C.byref(info)))
        obj = cls._from_handle(h, info.r_min, info.r_max)
        if adopt:
            obj._slab_owner = slab  # released after the tree (see __del__)
        return obj

    def __repr__(self) -> str:
        return (f"Capt(k={self.k}, n={self.n}, points={self.n_points}, "
                f"r_min={self.r_min}, r_max={self.r_max}, device=cuda:{self.device})")


def construct(cloud: PointCloud, params: BuildParams, use_rmin_shortcut: bool = True,
              device: int | None = None, stream=None) -> Capt:
    """Build a tree over ``cloud`` on the GPU (tree.py:139-241).

    Accepts a PointCloud, an (n, k) numpy array, or an (n, k) float32 CUDA
    tensor (device-resident build input)."""
    dev = _lib.default_device() if device is None else int(device)
    flags = 0
    if hasattr(cloud, "data_ptr") and getattr(cloud, "is_cuda", False):
        pts = cloud.contiguous()
        if pts.dtype.__repr__() != "torch.float32" or pts.ndim != 2:
            raise ValueError("device points must be an (n, k) float32 tensor")
        n0, k = int(pts.shape[0]), int(pts.shape[1])
        p = pts.data_ptr()
        keep = pts
        dev = pts.device.index if pts.device.index is not None else dev
    else:
        if not isinstance(cloud, PointCloud):
            cloud = PointCloud(cloud)
        keep = cloud.points
        n0, k = len(cloud), cloud.k
        p = keep.ctypes.data
        flags |= _lib.HOST_IO
    if n0 == 0:
        raise ValueError("cannot build a tree over an empty cloud")
    h = C.c_void_p()
    rc = _lib.lib().capt_tree_build(dev, k, p, n0, float(params.r_min), float(params.r_max),
                                    int(bool(use_rmin_shortcut)), flags,
                                    None if stream is None else int(stream), C.byref(h))
    _lib.check(rc, "capt_tree_build")
    del keep
    return Capt._from_handle(h, params.r_min, params.r_max)


def _centers_arg(tree: Capt, centers):
    """(device pointer or host array, flags, n, keepalive) for a centers array."""
    if hasattr(centers, "data_ptr") and getattr(centers, "is_cuda", False):
        import torch
        c = centers.contiguous()
        flags = 0
        if c.dtype == torch.float64:
            flags |= _lib.INPUT_F64
        elif c.dtype != torch.float32:
            c = c.to(torch.float32)
        return c.data_ptr(), flags, int(c.numel() // tree.k), c
    c = np.asarray(centers)
    if c.dtype == np.float32:
        c = np.ascontiguousarray(c)
        flags = _lib.HOST_IO
    else:
        c = np.ascontiguousarray(c, dtype=np.float64)
        flags = _lib.HOST_IO | _lib.INPUT_F64
    c = c.reshape(-1, tree.k)
    return c.ctypes.data, flags, len(c), c


def leaf_indices(tree: Capt, centers) -> np.ndarray:
    """Vectorised descent (tree.py:266-273) on the GPU."""
    p, flags, n, keep = _centers_arg(tree, centers)
    if flags & _lib.HOST_IO:
        out = np.empty(n, np.int64)
        optr = out.ctypes.data
    else:
        import torch
        out = torch.empty(n, dtype=torch.int64, device=keep.device)
        optr = out.data_ptr()
    if n:
        _lib.check(_lib.lib().capt_leaf_indices(tree.handle, p, n, flags, optr, None),
                   "capt_leaf_indices")
    return out


def leaf_index(tree: Capt, x) -> int:
    """Branch-free descent of one point (tree.py:244-251)."""
    return int(leaf_indices(tree, np.asarray(x, dtype=np.float64).reshape(1, tree.k))[0])


def leaf_index_counted(tree: Capt, x) -> tuple[int, int]:
    """As leaf_index plus the number of descent steps (always log2 n)."""
    return leaf_index(tree, x), tree.depth


def save_capt(tree: Capt, path) -> None:
    """Versioned little-endian binary dump, byte-identical format to
    tree.py:276-288 (32-bit floats)."""
    with open(path, "wb") as f:
        f.write(_HEADER.pack(MAGIC, tree.k, tree.n, tree.n_points,
                             np.float32(tree.r_min), np.float32(tree.r_max)))
        f.write(tree.tests.astype("<f4").tobytes())
        f.write(tree.aff_lo.astype("<f4").tobytes())
        f.write(tree.aff_hi.astype("<f4").tobytes())
        f.write(tree.offsets.astype("<i8").tobytes())
        f.write(tree.aff_values.astype("<f4").tobytes())


def load_capt(path, device: int | None = None) -> Capt:
    """Inverse of save_capt straight into device layout (tree.py:291-320).
    Like the reference, r_min/r_max come back as their fp32 values."""
    with open(path, "rb") as f:
        raw = f.read()
    if len(raw) < _HEADER.size:
        raise ValueError("truncated tree dump")
    magic, k, n, n_points, r_min, r_max = _HEADER.unpack_from(raw, 0)
    if magic != MAGIC:
        raise ValueError(f"bad magic {magic!r}; not a tree dump")
    pos = _HEADER.size

    def take(dtype, count):
        nonlocal pos
        arr = np.frombuffer(raw, dtype=dtype, count=count, offset=pos)
        pos += arr.nbytes
        return arr

    try:
        tests = take("<f4", n - 1)
        aff_lo = take("<f4", n * k).reshape(n, k)
        aff_hi = take("<f4", n * k).reshape(n, k)
        offsets = take("<i8", n + 1).astype(np.int64)
        values = take("<f4", int(offsets[-1]) * k)
    except ValueError as exc:
        raise ValueError(f"corrupt tree dump: {exc}") from exc
    if pos != len(raw):
        raise ValueError("trailing bytes in tree dump")
    return Capt(k=k, n_points=n_points, r_min=float(r_min), r_max=float(r_max),
                tests=tests, aff_lo=aff_lo, aff_hi=aff_hi, offsets=offsets,
                aff_values=values, device=device)
