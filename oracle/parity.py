"""Parity checks of the device path against the CPU oracle -- TEST
INFRASTRUCTURE ONLY (imported by tests/ and by bench.py after its timed
region; never by the product package).

* ``tree_parity``: a device tree vs ``oracle.construct`` on the same cloud
  (tree.py:139-241): ``tests``, ``offsets``, ``aff_lo``, ``aff_hi`` bit for
  bit (as uint32 patterns, so -0.0 / NaN cannot hide a difference) and the
  affordance sets in canonical per-leaf order.
* ``mask_parity``: packed verdict words vs ``oracle.collides_many``
  (query.py:184-219) or ``oracle.collides_groups`` (query.py:126-167), plus
  the number of boundary spheres -- some affordance-set point p of the
  sphere's leaf with |d^2(c, p) - r^2| < 1e-6 in float64 (SURVEY 8c parity
  contract; oracle scan_leaf) -- which the contract asks to report.
"""

from __future__ import annotations

import numpy as np

from . import oracle as O


def _bits(a) -> np.ndarray:
    a = np.ascontiguousarray(a)
    return a.view(np.uint32) if a.dtype == np.float32 else a


def tree_parity(dev_tree, cloud, r_min: float, r_max: float, use_rmin_shortcut: bool = True,
                ref=None) -> dict:
    """Compare ``dev_tree`` (anything ``oracle.tree_from`` accepts) with the
    oracle's construct of ``cloud``.  Returns a dict of per-array mismatch
    counts (all 0 on parity) and the oracle tree under ``"ref"``."""
    if ref is None:
        ref = O.construct(cloud, r_min, r_max, use_rmin_shortcut)
    got = O.tree_from(dev_tree)
    out = {"leaves": int(ref["n"]), "stored_points": int(ref["offsets"][-1])}
    if got["n"] != ref["n"] or got["k"] != ref["k"]:
        out.update(shape_mismatch=True, mismatches=1)
        return out
    mism = 0
    for key in ("tests", "offsets", "aff_lo", "aff_hi"):
        a, b = _bits(got[key]).ravel(), _bits(ref[key]).ravel()
        d = int(np.count_nonzero(a != b)) if a.shape == b.shape else max(a.size, b.size)
        out[key] = d
        mism += d
    if out["offsets"] == 0:
        a = _bits(O.canonical_values(got))
        b = _bits(O.canonical_values(ref))
        d = int(np.count_nonzero(a != b)) if a.shape == b.shape else max(a.size, b.size)
    else:
        d = -1  # sets not comparable
    out["aff_values_canonical"] = d
    mism += abs(d)
    out["mismatches"] = mism
    out["ties"] = int(ref.get("ties", 0))
    out["ref"] = ref
    return out


def unpack_words(words, n: int) -> np.ndarray:
    w = np.ascontiguousarray(words).view(np.uint32)
    return np.unpackbits(w.view(np.uint8), bitorder="little")[:n].astype(bool)


def mask_parity(tree, centers, radii, words, lane_width: int = 1, threads: int = 0,
                boundary: bool = True) -> dict:
    """Verdict words of ``len(radii) // lane_width`` groups against the
    oracle on ``tree`` (reference layout).  Returns {"spheres", "units",
    "mismatches", "collisions", "boundary"}."""
    c = np.asarray(centers)
    r = np.asarray(radii)
    n = len(r)
    L = int(lane_width)
    got = unpack_words(words, n // L)
    if L == 1:
        exp, cnt = O.collides_many(tree, c, r, threads=threads, return_counters=True)
        bnd = cnt[1]
    else:
        exp = O.collides_groups(tree, c, r, L, threads=threads)
        bnd = None
        if boundary:  # per-sphere scan of every lane (counted over all spheres)
            _, cnt = O.collides_many(tree, c, r, threads=threads, return_counters=True)
            bnd = cnt[1]
    bad = np.nonzero(got != exp)[0]
    return {"spheres": int(n), "units": int(n // L), "mismatches": int(len(bad)),
            "first_mismatch": int(bad[0]) if len(bad) else None,
            "collisions": int(exp.sum()), "boundary": bnd}
