"""Query traces and their replay on the device.

A trace is the reference's CSV of query batches (io.py:98-165): header
``batch,x,y,z,r[,expected]``; rows sharing a batch id form one record, whose
optional expected flag is the OR over its spheres.  ``capt_verdicts`` replays
every record of a trace in ONE device call (bench.py:43-107 semantics: the
any-collision verdict per record), ``verify_trace`` checks the expected
column (bench.py:110-116) and ``query_phase`` times the replay split by
workload class (bench.py:172-199).

Replay layout: records are padded to a common power-of-two lane width
(<= 32); longer records take several consecutive lane groups whose verdicts
are OR-ed on the host; padding lanes are masked.  The band check raises the
reference's ValueError for the first out-of-band radius in trace order.
"""

from __future__ import annotations

import csv
import time
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .tree import Capt

__all__ = ["ParseError", "VerificationError", "QueryTraceRecord", "read_trace", "write_trace",
           "capt_verdicts", "verify_trace", "query_phase"]

_COLUMNS = ["batch", "x", "y", "z", "r"]


class ParseError(ValueError):
    """Malformed trace file; the message starts with ``path:line:``."""

    def __init__(self, path, line: int, message: str):
        super().__init__(f"{path}:{line}: {message}")
        self.path = path
        self.line = line


class VerificationError(Exception):
    """A replayed verdict disagreed with the trace's expected column."""


@dataclass
class QueryTraceRecord:
    batch_id: int
    centers: np.ndarray  # (m, 3) float32
    radii: np.ndarray    # (m,) float32
    expected: Optional[bool] = None

    def __len__(self) -> int:
        return len(self.radii)


def _expected(text: str, path, line: int) -> Optional[bool]:
    t = text.strip().lower()
    if t == "":
        return None
    if t in ("1", "true"):
        return True
    if t in ("0", "false"):
        return False
    raise ParseError(path, line, f"bad expected value {text!r}")


def read_trace(path) -> list[QueryTraceRecord]:
    """Parse a trace (io.py:98-146): same header rule, the same checks
    (field count, numeric and finite values, r > 0, one expected flag per
    batch) and the same record order (first appearance of each batch id)."""
    batches: dict[int, list] = {}
    with open(path, "r", encoding="utf-8", errors="replace", newline="") as f:
        rows = csv.reader(f)
        header = next(rows, None)
        if header is None:
            raise ParseError(path, 1, "empty trace file")
        header = [h.strip().lower() for h in header]
        if header not in (_COLUMNS, _COLUMNS + ["expected"]):
            raise ParseError(path, 1, f"bad header {header!r}")
        width = len(header)
        for line, row in enumerate(rows, start=2):
            if not row or (len(row) == 1 and not row[0].strip()):
                continue
            if len(row) != width:
                raise ParseError(path, line, f"expected {width} fields, got {len(row)}")
            try:
                bid = int(row[0])
                x, y, z, r = (float(v) for v in row[1:5])
            except ValueError:
                raise ParseError(path, line, f"bad numeric field in {row!r}") from None
            if not np.all(np.isfinite([x, y, z, r])):
                raise ParseError(path, line, "non-finite value")
            if r <= 0:
                raise ParseError(path, line, f"radius must be > 0, got {r}")
            exp = _expected(row[5], path, line) if width == 6 else None
            rec = batches.get(bid)
            if rec is None:
                batches[bid] = [[(x, y, z)], [r], exp]
            else:
                if rec[2] != exp:
                    raise ParseError(path, line, f"inconsistent expected flag in batch {bid}")
                rec[0].append((x, y, z))
                rec[1].append(r)
    return [QueryTraceRecord(bid, np.asarray(c, np.float32), np.asarray(r, np.float32), e)
            for bid, (c, r, e) in batches.items()]


def write_trace(records: list[QueryTraceRecord], path) -> None:
    """Inverse of read_trace (io.py:149-161); float32 values are written as the
    shortest decimal that round-trips."""
    with_exp = any(rec.expected is not None for rec in records)
    with open(path, "w", encoding="utf-8", newline="") as f:
        w = csv.writer(f)
        w.writerow(_COLUMNS + (["expected"] if with_exp else []))
        for rec in records:
            tail = [] if not with_exp else ["" if rec.expected is None else str(int(rec.expected))]
            for c, r in zip(rec.centers, rec.radii):
                w.writerow([str(rec.batch_id)] + [str(np.float32(v)) for v in c[:3]]
                           + [str(np.float32(r))] + tail)


def _pack(records: list[QueryTraceRecord]):
    """Records -> (centers, radii, lane mask, lane width, group -> record)."""
    longest = max((len(r) for r in records), default=1)
    width = 1
    while width < min(longest, 32):
        width *= 2
    groups = [max(1, -(-len(r) // width)) for r in records]
    n = sum(groups) * width
    centers = np.zeros((n, 3), np.float32)
    radii = np.zeros(n, np.float32)
    mask = np.zeros(n, np.uint8)
    owner = np.repeat(np.arange(len(records)), groups)
    pos = 0
    for rec, g in zip(records, groups):
        m = len(rec)
        centers[pos:pos + m] = rec.centers
        radii[pos:pos + m] = rec.radii
        mask[pos:pos + m] = 1
        pos += g * width
    return centers, radii, mask, width, owner


def capt_verdicts(tree: Capt, records: list[QueryTraceRecord],
                  use_aabb_prefilter: bool = True) -> np.ndarray:
    """Any-collision verdict of every record (bench.py:43-107), one device
    call for the whole trace."""
    from . import _lib
    from .query import _host_query

    out = np.zeros(len(records), dtype=bool)
    if not records:
        return out
    centers, radii, mask, width, owner = _pack(records)
    # the band check in trace order (the reference checks the float64 upcast)
    for rec in records:
        bad = (rec.radii.astype(np.float64) < tree.r_min) | (rec.radii.astype(np.float64) > tree.r_max)
        if bad.any():
            r = float(rec.radii[np.nonzero(bad)[0][0]])
            raise ValueError(f"radius {r} outside the tree's exactness band "
                             f"[{tree.r_min}, {tree.r_max}]")
    bits, _, _ = _host_query(tree, centers, radii, 0, width, mask, use_aabb_prefilter, False,
                             mode=0)
    np.logical_or.at(out, owner, bits)
    return out


def verify_trace(records: list[QueryTraceRecord], verdicts: np.ndarray) -> None:
    """Raise VerificationError naming the first batch whose verdict disagrees
    with its expected flag (bench.py:110-116)."""
    for rec, got in zip(records, verdicts):
        if rec.expected is not None and bool(got) != rec.expected:
            raise VerificationError(f"batch {rec.batch_id}: expected {rec.expected}, "
                                    f"got {bool(got)}")


def query_phase(tree: Capt, records: list[QueryTraceRecord], use_aabb_prefilter: bool = True,
                repetitions: int = 3) -> dict:
    """Median wall time per sphere (ns) of the replay for all records and for
    the colliding / non-colliding subsets (bench.py:172-199), host buffers
    in and verdicts out, one warm-up call each."""

    def ns_per_sphere(recs):
        if not recs:
            return None
        capt_verdicts(tree, recs, use_aabb_prefilter)
        times = []
        for _ in range(max(1, repetitions)):
            t0 = time.perf_counter()
            capt_verdicts(tree, recs, use_aabb_prefilter)
            times.append(time.perf_counter() - t0)
        return float(np.median(times)) * 1e9 / sum(len(r) for r in recs)

    return {
        "query_ns_all": ns_per_sphere(records),
        "query_ns_colliding": ns_per_sphere([r for r in records if r.expected is True]),
        "query_ns_non_colliding": ns_per_sphere([r for r in records if r.expected is False]),
    }
