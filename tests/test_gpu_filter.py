"""Device Morton/Z-order filter (capt_filter_cloud) vs the reference's outputs
(golden fixtures) and the oracle: bit-exact point arrays, same order."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2406_02807_b200")
from paper_2406_02807_b200 import workloads as W  # noqa: E402


def test_filter_matches_reference_golden():
    z = load_golden("filters.npz")
    for name in z["names"]:
        pts = z[f"{name}/points"]
        r = float(z[f"{name}/r"][0])
        if f"{name}/base" in z:
            cfg = P.FilterConfig(r, base=z[f"{name}/base"], max_reach=float(z[f"{name}/max_reach"][0]))
        else:
            cfg = P.FilterConfig(r)
        got = P.filter_cloud(P.PointCloud(pts), cfg).points
        assert np.array_equal(got, z[f"{name}/out"]), name


def test_filter_cfg2_full_vs_oracle():
    raw = W.cfg2_raw_cloud()
    got = P.filter_cloud(P.PointCloud(raw), P.FilterConfig(0.01)).points
    exp = O.filter_cloud(raw, 0.01)
    assert np.array_equal(got, exp)
    assert 10000 < len(got) < len(raw)


@pytest.mark.parametrize("r", [0.0, 0.005, 0.05, 0.3])
def test_filter_random_radii(r):
    rng = np.random.default_rng(int(r * 1000) + 1)
    pts = rng.uniform(-1, 1, (20000, 3)).astype(np.float32)
    pts[:500] = pts[500:1000]  # duplicates
    assert np.array_equal(P.filter_cloud(P.PointCloud(pts), P.FilterConfig(r)).points,
                          O.filter_cloud(pts, r))


def test_filter_k2_k1_and_edge_cases():
    rng = np.random.default_rng(3)
    for k in (1, 2):
        pts = rng.uniform(0, 1, (3000, k)).astype(np.float32)
        assert np.array_equal(P.filter_cloud(P.PointCloud(pts), P.FilterConfig(0.01)).points,
                              O.filter_cloud(pts, 0.01))
    empty = P.PointCloud(np.empty((0, 3), np.float32))
    assert len(P.filter_cloud(empty, P.FilterConfig(0.1))) == 0
    one = P.PointCloud(np.array([[1, 2, 3]], np.float32))
    assert np.array_equal(P.filter_cloud(one, P.FilterConfig(0.1)).points, one.points)
    two = np.array([[0, 0, 0], [1, 0, 0]], np.float32)
    assert len(P.filter_cloud(P.PointCloud(two), P.FilterConfig(2.0))) == 1
    # degenerate axis (planar cloud)
    plane = rng.uniform(0, 1, (5000, 3)).astype(np.float32)
    plane[:, 2] = 0.5
    assert np.array_equal(P.filter_cloud(P.PointCloud(plane), P.FilterConfig(0.02)).points,
                          O.filter_cloud(plane, 0.02))


def test_reach_filter():
    pts = np.array([[0.5, 0, 0], [2, 0, 0], [0, 1, 0]], dtype=np.float32)
    out = P.reach_filter(P.PointCloud(pts), np.zeros(3), 1.0)
    assert np.array_equal(out.points, pts[[0, 2]])
    rng = np.random.default_rng(21)
    cloud = rng.uniform(-1, 1, (5000, 3)).astype(np.float32)
    base = np.array([0.1, -0.2, 0.3])
    out = P.reach_filter(P.PointCloud(cloud), base, 0.7)
    d = ((cloud.astype(np.float64) - base) ** 2).sum(1)
    assert np.array_equal(out.points, cloud[d <= 0.49])
    cfg = P.FilterConfig(0.05, base=base, max_reach=0.7)
    assert np.array_equal(P.filter_cloud(P.PointCloud(cloud), cfg).points,
                          O.filter_cloud(cloud, 0.05, base=base, max_reach=0.7))
    far = P.PointCloud(np.full((4, 3), 9.0, dtype=np.float32))
    assert len(P.filter_cloud(far, P.FilterConfig(0.05, base=np.zeros(3), max_reach=1.0))) == 0


def test_filter_then_build_pipeline():
    raw = W.cfg2_raw_cloud()
    filt = P.filter_cloud(P.PointCloud(raw), P.FilterConfig(0.01))
    tree = P.construct(filt, P.BuildParams(0.01, 0.08))
    ref = O.construct(filt.points, 0.01, 0.08)
    assert np.array_equal(tree.offsets, ref["offsets"])
    assert np.array_equal(O.canonical_values(tree), O.canonical_values(ref))
    c, r = W.cfg2_queries(filt.points, n=1 << 18)
    assert np.array_equal(P.collides_many(tree, c, r), O.collides_many(ref, c, r))
