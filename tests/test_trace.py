"""Query traces (the reference's io.py:98-165 CSV) and their device replay
(bench.py:43-199 semantics), against fixtures produced by the reference's own
generator, writer and replay (tests/golden/make_golden.py:make_trace)."""

import numpy as np
import pytest

from conftest import load_golden

from paper_2406_02807_b200 import trace as T

CASES = ("b8", "b5", "b40")


def _write(tmp_path, name, data):
    p = tmp_path / name
    p.write_bytes(data)
    return str(p)


@pytest.mark.parametrize("case", CASES)
def test_read_write_round_trip(tmp_path, case):
    z = load_golden("trace.npz")
    raw = bytes(z[f"{case}/csv"])
    path = _write(tmp_path, "t.csv", raw)
    recs = T.read_trace(path)
    assert [r.batch_id for r in recs] == list(z[f"{case}/batch_ids"])
    assert [len(r) for r in recs] == list(z[f"{case}/sizes"])
    assert [-1 if r.expected is None else int(r.expected) for r in recs] == \
        list(z[f"{case}/expected"])
    assert all(r.centers.dtype == np.float32 and r.radii.dtype == np.float32 for r in recs)
    out = tmp_path / "back.csv"
    T.write_trace(recs, str(out))
    assert out.read_bytes() == raw  # byte-identical to the reference's writer


@pytest.mark.parametrize("body, line, text", [
    (b"", 1, "empty trace file"),
    (b"batch,x,y,z\n", 1, "bad header"),
    (b"batch,x,y,z,r\n0,1,2,3\n", 2, "expected 5 fields, got 4"),
    (b"batch,x,y,z,r\n0,1,2,a,0.1\n", 2, "bad numeric field"),
    (b"batch,x,y,z,r\n0,1,2,inf,0.1\n", 2, "non-finite value"),
    (b"batch,x,y,z,r\n0,1,2,3,0\n", 2, "radius must be > 0"),
    (b"batch,x,y,z,r,expected\n0,1,2,3,0.1,1\n\n0,1,2,3,0.1,0\n", 4,
     "inconsistent expected flag in batch 0"),
    (b"batch,x,y,z,r,expected\n0,1,2,3,0.1,maybe\n", 2, "bad expected value"),
])
def test_parse_errors(tmp_path, body, line, text):
    path = _write(tmp_path, "bad.csv", body)
    with pytest.raises(T.ParseError) as e:
        T.read_trace(path)
    assert e.value.line == line and str(e.value).startswith(f"{path}:{line}: ")
    assert text in str(e.value)


def test_blank_lines_and_optional_expected(tmp_path):
    path = _write(tmp_path, "ok.csv",
                  b"Batch, X ,y,z,R\n3,0,0,0,0.05\n\n1,1,1,1,0.02\n3,0.5,0,0,0.04\n")
    recs = T.read_trace(path)
    assert [r.batch_id for r in recs] == [3, 1] and [len(r) for r in recs] == [2, 1]
    assert all(r.expected is None for r in recs)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_device_replay_matches_reference(tmp_path, case):
    import paper_2406_02807_b200 as P
    z = load_golden("trace.npz")
    lo, hi = z["band"]
    tree = P.construct(P.PointCloud(z["points"]), P.BuildParams(float(lo), float(hi)))
    recs = T.read_trace(_write(tmp_path, "t.csv", bytes(z[f"{case}/csv"])))
    got = T.capt_verdicts(tree, recs)
    assert np.array_equal(got, z[f"{case}/verdicts"])
    assert np.array_equal(T.capt_verdicts(tree, recs, use_aabb_prefilter=False),
                          z[f"{case}/nopre"])
    T.verify_trace(recs, got)
    recs[3].expected = not recs[3].expected
    with pytest.raises(T.VerificationError, match=f"batch {recs[3].batch_id}: expected"):
        T.verify_trace(recs, got)
    rep = T.query_phase(tree, recs[:20], repetitions=1)
    assert rep["query_ns_all"] > 0
    recs[5].radii[0] = np.float32(0.5)
    with pytest.raises(ValueError, match="outside the tree's exactness band"):
        T.capt_verdicts(tree, recs)
