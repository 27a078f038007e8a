"""ctypes wrapper over the CPU oracle (liboracle.so) -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline /
``--impl reference`` legs import this module.  It restates the reference
package ``captree`` (/root/reference/pkg/src/captree) in C; each wrapper names
the reference function it stands in for.  The restatement is pinned against
the reference itself by tests/test_oracle_golden.py (fixtures produced by
tests/golden/make_golden.py while importing the real reference).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc, no FMA contraction)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        build()
    L = C.CDLL(_LIB_PATH)
    i64 = C.c_int64
    L.oracle_construct.restype = C.c_void_p
    L.oracle_construct.argtypes = [C.c_int, i64, _f32p, C.c_double, C.c_double,
                                   C.c_int, C.POINTER(i64)]
    L.oracle_tree_sizes.argtypes = [C.c_void_p, C.POINTER(i64), C.POINTER(i64)]
    L.oracle_tree_export.argtypes = [C.c_void_p, _f32p, _f32p, _f32p, _i64p, _f32p]
    L.oracle_tree_free.argtypes = [C.c_void_p]
    L.oracle_canonicalize.argtypes = [C.c_int, i64, _i64p, _f32p]
    L.oracle_leaf_indices.argtypes = [C.c_int, i64, _f32p, _f64p, i64, _i64p]
    L.oracle_collides_many.argtypes = [C.c_int, i64, _f32p, _f32p, _f32p, _i64p,
                                       _f32p, _f64p, _f64p, i64, C.c_int, _u8p,
                                       C.c_void_p, C.c_int]
    L.oracle_collides_groups.argtypes = [C.c_int, i64, _f32p, _f32p, _f32p, _i64p,
                                         _f32p, _f64p, _f64p, C.c_void_p, i64,
                                         C.c_int, C.c_int, _u8p, _i64p, C.c_int]
    L.oracle_brute_collides_many.argtypes = [C.c_int, i64, _f32p, _f64p, _f64p,
                                             i64, _u8p, C.c_int]
    L.oracle_filter_cloud.restype = i64
    L.oracle_filter_cloud.argtypes = [C.c_int, i64, _f32p, C.c_double, C.c_int,
                                      _f64p, C.c_double, _f32p]
    L.oracle_morton_keys.argtypes = [C.c_int, i64, _f32p, _f64p, _f64p, _i32p, _u64p]
    _lib = L
    return L


def _c32(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a if shape is None else a.reshape(shape)


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def construct(points, r_min: float, r_max: float, use_rmin_shortcut: bool = True) -> dict:
    """Stand-in for captree.construct (tree.py:139-241). Returns the Capt arrays
    (reference layout) plus ``ties`` = straddling-tie split count."""
    pts = _c32(points)
    if pts.ndim != 2 or len(pts) == 0:
        raise ValueError("cannot build a tree over an empty cloud")
    k = pts.shape[1]
    ties = C.c_int64(0)
    h = lib().oracle_construct(k, len(pts), pts.ravel(), float(r_min), float(r_max),
                               int(bool(use_rmin_shortcut)), C.byref(ties))
    if not h:
        raise ValueError("oracle_construct failed")
    n = C.c_int64()
    tot = C.c_int64()
    lib().oracle_tree_sizes(h, C.byref(n), C.byref(tot))
    n, tot = n.value, tot.value
    tests = np.empty(max(n - 1, 1), np.float32)
    lo = np.empty((n, k), np.float32)
    hi = np.empty((n, k), np.float32)
    off = np.empty(n + 1, np.int64)
    vals = np.empty(max(tot * k, 1), np.float32)
    lib().oracle_tree_export(h, tests, lo, hi, off, vals)
    lib().oracle_tree_free(h)
    return dict(k=k, n=n, n_points=len(pts), r_min=float(r_min), r_max=float(r_max),
                depth=int(n).bit_length() - 1, tests=tests[: n - 1].copy(),
                aff_lo=lo, aff_hi=hi, offsets=off, aff_values=vals[: tot * k].copy(),
                ties=int(ties.value))


def tree_from(obj) -> dict:
    """Reference-layout dict from a captree.Capt / our Capt / a dict."""
    if isinstance(obj, dict):
        return obj
    return dict(k=obj.k, n=obj.n, n_points=obj.n_points, r_min=obj.r_min,
                r_max=obj.r_max, depth=obj.depth,
                tests=np.asarray(obj.tests, np.float32),
                aff_lo=np.asarray(obj.aff_lo, np.float32),
                aff_hi=np.asarray(obj.aff_hi, np.float32),
                offsets=np.asarray(obj.offsets, np.int64),
                aff_values=np.asarray(obj.aff_values, np.float32))


def canonical_values(tree) -> np.ndarray:
    """aff_values in canonical per-leaf order."""
    t = tree_from(tree)
    vals = np.array(t["aff_values"], dtype=np.float32, copy=True)
    if vals.size == 0:
        return vals
    lib().oracle_canonicalize(t["k"], t["n"], _i64p_arr(t["offsets"]), vals)
    return vals


def _i64p_arr(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _tree_args(t):
    vals = t["aff_values"]
    if vals.size == 0:
        vals = np.zeros(1, np.float32)
    tests = t["tests"] if len(t["tests"]) else np.zeros(1, np.float32)
    return (t["k"], t["n"], _c32(tests), _c32(t["aff_lo"]).ravel(),
            _c32(t["aff_hi"]).ravel(), _i64p_arr(t["offsets"]), _c32(vals))


def leaf_indices(tree, centers) -> np.ndarray:
    """Stand-in for tree.leaf_indices (tree.py:266-273)."""
    t = tree_from(tree)
    c = _c64(centers).reshape(-1, t["k"])
    out = np.empty(len(c), np.int64)
    tests = t["tests"] if len(t["tests"]) else np.zeros(1, np.float32)
    lib().oracle_leaf_indices(t["k"], t["n"], _c32(tests), c.ravel(), len(c), out)
    return out


def collides_many(tree, centers, radii, use_aabb_prefilter: bool = True,
                  threads: int = 0, return_counters: bool = False):
    """Stand-in for query.collides_many (query.py:184-219) without the radius
    check.  counters = (collisions, boundary spheres, points scanned)."""
    t = tree_from(tree)
    c = _c64(centers).reshape(-1, t["k"])
    r = _c64(radii).ravel()
    out = np.empty(len(c), np.uint8)
    cnt = np.zeros(3, np.int64)
    lib().oracle_collides_many(*_tree_args(t), c.ravel(), r, len(c),
                               int(bool(use_aabb_prefilter)), out,
                               cnt.ctypes.data if return_counters else None, int(threads))
    res = out.astype(bool)
    return (res, tuple(int(x) for x in cnt)) if return_counters else res


def collides_groups(tree, centers, radii, lane_width: int = 8, mask=None,
                    use_aabb_prefilter: bool = True, threads: int = 0,
                    return_counters: bool = False):
    """Stand-in for collides_batch(...).any_collision over consecutive groups
    (query.py:126-167; bench.capt_verdicts batch mode bench.py:54-85).
    counters = (colliding groups, aabb rejections, points scanned)."""
    t = tree_from(tree)
    c = _c64(centers).reshape(-1, t["k"])
    r = _c64(radii).ravel()
    if len(c) % lane_width:
        raise ValueError("sphere count must be a multiple of lane_width")
    ng = len(c) // lane_width
    out = np.empty(ng, np.uint8)
    cnt = np.zeros(3, np.int64)
    m = None
    if mask is not None:
        m = np.ascontiguousarray(mask, dtype=np.uint8).ravel()
    lib().oracle_collides_groups(*_tree_args(t), c.ravel(), r,
                                 m.ctypes.data if m is not None else None, ng,
                                 int(lane_width), int(bool(use_aabb_prefilter)),
                                 out, cnt, int(threads))
    res = out.astype(bool)
    return (res, tuple(int(x) for x in cnt)) if return_counters else res


def brute_collides_many(points, centers, radii, threads: int = 0) -> np.ndarray:
    """Stand-in for oracle.brute_collides_many (oracle.py:34-49)."""
    p = _c32(points)
    k = p.shape[1]
    c = _c64(centers).reshape(-1, k)
    r = _c64(radii).ravel()
    out = np.empty(len(c), np.uint8)
    if len(p) == 0:
        return np.zeros(len(c), bool)
    lib().oracle_brute_collides_many(k, len(p), p.ravel(), c.ravel(), r, len(c), out,
                                     int(threads))
    return out.astype(bool)


def filter_cloud(points, r_filter: float, base=None, max_reach: Optional[float] = None):
    """Stand-in for morton.filter_cloud (morton.py:185-236)."""
    p = _c32(points)
    k = p.shape[1]
    out = np.empty((max(len(p), 1), k), np.float32)
    has = base is not None
    b = _c64(base if has else np.zeros(k))
    n = lib().oracle_filter_cloud(k, len(p), p.ravel() if len(p) else np.zeros(1, np.float32),
                                  float(r_filter), int(has), b,
                                  float(max_reach) if has else 0.0, out.reshape(-1))
    return out[:n].copy()


def morton_keys(points, lo, hi, perm) -> np.ndarray:
    """Stand-in for morton.morton_keys (morton.py:113-126)."""
    p = _c32(points)
    k = p.shape[1]
    keys = np.empty(len(p), np.uint64)
    lib().oracle_morton_keys(k, len(p), p.ravel(), _c64(lo), _c64(hi),
                             np.ascontiguousarray(perm, dtype=np.int32), keys)
    return keys
