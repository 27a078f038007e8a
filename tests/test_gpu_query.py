"""Parity of the CUDA query path (through the C-ABI) with the oracle and with
reference-generated golden masks.  Trees here are uploaded from the
reference/oracle layout so the query kernels are tested independently of the
device build (tests/test_gpu_build.py covers construct)."""

import numpy as np
import pytest

from conftest import golden_tree, load_golden
from oracle import oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2406_02807_b200")


def upload(t):
    return P.Capt(t["k"], t["n_points"], t["r_min"], t["r_max"], t["tests"], t["aff_lo"],
                  t["aff_hi"], t["offsets"], t["aff_values"])


def unpack(b, n):
    return np.unpackbits(b)[:n].astype(bool)


def test_golden_masks_and_groups():
    z = load_golden("queries.npz")
    for name in z["names"]:
        pts = z[f"{name}/points"]
        rmin, rmax = z[f"{name}/band"]
        tree = upload(O.construct(pts, rmin, rmax))
        c, r = z[f"{name}/centers"], z[f"{name}/radii"]
        n = len(r)
        assert np.array_equal(P.collides_many(tree, c, r), unpack(z[f"{name}/mask"], n)), name
        assert np.array_equal(P.collides_many(tree, c, r, use_aabb_prefilter=False),
                              unpack(z[f"{name}/mask_nopre"], n)), name
        # float64 inputs (exact upcasts) take the same path
        assert np.array_equal(P.collides_many(tree, c.astype(np.float64), r.astype(np.float64)),
                              unpack(z[f"{name}/mask"], n)), name
        assert np.array_equal(P.leaf_indices(tree, c), z[f"{name}/leaf"]), name
        lane = unpack(z[f"{name}/lane_mask"], n)
        gb = unpack(z[f"{name}/group8"], n // 8)
        scanned = z[f"{name}/group8_scanned"]
        c64, r64 = c.astype(np.float64), r.astype(np.float64)
        for g in range(0, n // 8, 97):
            s = slice(8 * g, 8 * g + 8)
            out = P.collides_batch(tree, P.SphereBatch(c64[s], r64[s], lane[s]),
                                   collect_stats=True)
            assert out.any_collision == gb[g], (name, g)
            assert out.points_scanned == scanned[g], (name, g)


def test_cfg0_golden_slice():
    from paper_2406_02807_b200 import workloads as W
    z = load_golden("cfg0.npz")
    tree = upload(golden_tree(z, ""))
    n = int(z["n_queries"][0])
    c, r = W.cfg0_queries()
    got = P.collides_many(tree, c[:n], r[:n])
    assert np.array_equal(got, unpack(z["mask"], n))


def test_hand_cases():
    z = load_golden("hand.npz")
    tree = upload(golden_tree(z, "tiny/"))
    got = P.collides_many(tree, z["tiny/centers"], z["tiny/radii"])
    assert list(got) == [True, False, True, True, False, True]
    assert P.collides(tree, P.Sphere(np.array([0.0, 0.0, 0.05]), 0.1))
    assert not P.collides(tree, P.Sphere(np.array([0.5, 0.5, 0.5]), 0.5))
    assert P.collides(tree, P.Sphere(np.array([2.0, 0.0, 0.0]), 1.0))  # tangency
    c = np.array([1.5, 0.0, 0.0])
    assert P.collides(tree, P.Sphere(c, 0.5))
    assert not P.collides(tree, P.Sphere(c, np.nextafter(0.5, 0.0)))
    assert P.collides(tree, P.Sphere(c, np.nextafter(0.5, 1.0)))
    with pytest.raises(ValueError, match="exactness band"):
        P.collides(tree, P.Sphere(np.zeros(3) + 5.0, 0.001))
    with pytest.raises(ValueError):
        P.collides(tree, P.Sphere(np.zeros(3) + 5.0, 3.0))
    assert not P.collides_unchecked(tree, P.Sphere(np.full(3, 5.0), 0.001))


def test_radius_check_and_unchecked():
    z = load_golden("hand.npz")
    tree = upload(golden_tree(z, "tiny/"))
    centers = np.zeros((2, 3))
    with pytest.raises(ValueError, match=r"radius 5.0 outside the tree's exactness band \[0.01, 2.0\]"):
        P.collides_many(tree, centers, np.array([0.5, 5.0]))
    out = P.collides_many(tree, centers, np.array([0.5, 5.0]), check_radii=False)
    assert out.all()
    # empty input
    assert P.collides_many(tree, np.zeros((0, 3), np.float32), np.zeros(0, np.float32)).shape == (0,)


def test_float64_inputs_not_fp32_exact():
    rng = np.random.default_rng(17)
    pts = rng.uniform(0, 1, (300, 3)).astype(np.float32)
    t = O.construct(pts, 0.01, 0.08)
    tree = upload(t)
    c = rng.uniform(-0.1, 1.1, (20000, 3))
    r = rng.uniform(0.01, 0.08, 20000)
    # tangency spheres in float64 (not representable in fp32)
    p = pts.astype(np.float64)[rng.integers(0, 300, 5000)]
    d = rng.normal(size=(5000, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    rr = rng.uniform(0.01, 0.08, 5000)
    c = np.concatenate([c, p + d * rr[:, None]])
    r = np.concatenate([r, rr])
    got = P.collides_many(tree, c, r)
    assert np.array_equal(got, O.collides_many(t, c, r))
    assert np.array_equal(got, O.brute_collides_many(pts, c, r))


def test_nonfinite_and_extreme_inputs():
    rng = np.random.default_rng(3)
    pts = rng.uniform(0, 1, (100, 3)).astype(np.float32)  # padded to 128 leaves
    t = O.construct(pts, 0.01, 0.08)
    tree = upload(t)
    c = rng.uniform(-0.2, 1.2, (64, 3))
    c[0, 0] = np.nan
    c[1, 1] = np.inf
    c[2, 2] = -np.inf
    c[3] = 1e30
    r = rng.uniform(0.01, 0.08, 64)
    r[4] = np.nan
    r[5] = 0.0
    r[6] = 1e30
    r[7] = -0.05
    r[8] = np.inf
    for pre in (True, False):
        got = P.collides_many(tree, c, r, use_aabb_prefilter=pre, check_radii=False)
        exp = O.collides_many(t, c, r, use_aabb_prefilter=pre)
        assert np.array_equal(got, exp), pre


def test_random_parity_large_with_counters():
    from paper_2406_02807_b200 import workloads as W
    cloud = W.cfg1_cloud()
    t = O.construct(cloud, 0.02, 0.08)
    tree = upload(t)
    c, r = W.cfg1_queries(cloud, n_groups=1 << 17)
    exp, ecnt = O.collides_many(t, c, r, return_counters=True)
    assert np.array_equal(P.collides_many(tree, c, r), exp)
    # per-sphere counters: collisions, boundary spheres, points scanned
    from paper_2406_02807_b200.query import _host_query
    bits, cnt, _ = _host_query(tree, c, r, 0, 1, None, True, True, stats=True)
    assert np.array_equal(bits, exp)
    assert int(cnt[0]) == ecnt[0] and int(cnt[1]) == ecnt[1] and int(cnt[2]) == ecnt[2]
    # groups of 8 with early exit: bits + sequential points_scanned + rejections
    gexp, gcnt = O.collides_groups(t, c, r, 8, return_counters=True)
    gbits, _, _ = _host_query(tree, c, r, 0, 8, None, True, True)
    assert np.array_equal(gbits, gexp)
    gbits, cnt, _ = _host_query(tree, c, r, 0, 8, None, True, True, stats=True)
    assert np.array_equal(gbits, gexp)
    assert int(cnt[0]) == gcnt[0] and int(cnt[4]) == gcnt[1] and int(cnt[2]) == gcnt[2]
    # other lane widths
    for L in (1, 2, 4, 16, 32):
        gb, _, _ = _host_query(tree, c, r, 0, L, None, True, True)
        assert np.array_equal(gb, exp.reshape(-1, L).any(1)), L


def test_lane_masks_and_collides_any():
    z = load_golden("hand.npz")
    tree = upload(golden_tree(z, "tiny/"))
    miss = P.Sphere(np.array([5.0, 5.0, 5.0]), 0.5)
    hit = P.Sphere(np.array([0.0, 0.0, 0.1]), 0.5)
    assert not P.collides_any(tree, [])
    assert not P.collides_any(tree, [miss] * 20)
    assert P.collides_any(tree, [miss] * 17 + [hit])
    assert P.collides_any(tree, [hit] + [miss] * 17)
    centers = np.tile(np.array([5.0, 5.0, 5.0]), (4, 1))
    radii = np.array([0.5, 99.0, 0.5, 0.5])
    mask = np.array([True, False, True, True])
    assert not P.collides_batch(tree, P.SphereBatch(centers, radii, mask)).any_collision
    with pytest.raises(ValueError):
        P.collides_batch(tree, P.SphereBatch(centers, radii, np.ones(4, bool)))
    far = np.tile(np.array([50.0, 50.0, 50.0]), (8, 1))
    out = P.collides_batch(tree, P.SphereBatch(far, np.full(8, 0.5), np.ones(8, bool)),
                           collect_stats=True)
    assert not out.any_collision and out.aabb_rejections == 8 and out.points_scanned == 0


def test_batch_lane_bits_match_scalar():
    rng = np.random.default_rng(31)
    pts = rng.uniform(0, 1, (256, 3)).astype(np.float32)
    t = O.construct(pts, 0.01, 0.08)
    tree = upload(t)
    for L in (1, 2, 8, 16, 64):
        for _ in range(20):
            c = rng.uniform(-0.1, 1.1, (L, 3))
            r = rng.uniform(0.01, 0.08, L)
            m = rng.uniform(size=L) < 0.8
            out = P.collides_batch(tree, P.SphereBatch(c, r, m), want_lane_bits=True)
            exp = O.collides_many(t, c, r) & m
            assert np.array_equal(out.lane_bits, exp)
            assert out.any_collision == exp.any()
            g = P.collides_batch(tree, P.SphereBatch(c, r, m), collect_stats=True)
            eg, ec = O.collides_groups(t, c, r, L, mask=m, return_counters=True)
            assert g.any_collision == eg[0]
            assert g.points_scanned == ec[2] and g.aabb_rejections == ec[1]


def test_export_and_save_load(tmp_path):
    z = load_golden("trees.npz")
    for name in z["names"]:
        t = golden_tree(z, f"{name}/")
        tree = upload(t)
        assert np.array_equal(tree.tests, t["tests"])
        assert np.array_equal(tree.offsets, t["offsets"])
        assert np.array_equal(tree.aff_lo, t["aff_lo"])
        assert np.array_equal(tree.aff_hi, t["aff_hi"])
        assert np.array_equal(tree.aff_values, t["aff_values"])
        p = tmp_path / f"{name}.capt"
        P.save_capt(tree, p)
        back = P.load_capt(p)
        assert np.array_equal(back.aff_values, t["aff_values"])
        assert np.float32(back.r_min) == np.float32(t["r_min"])


def test_device_tensor_path():
    import torch
    rng = np.random.default_rng(5)
    pts = rng.uniform(-1, 1, (2048, 3)).astype(np.float32)
    t = O.construct(pts, 0.01, 0.08)
    tree = upload(t)
    c = rng.uniform(-1.1, 1.1, (100000, 3)).astype(np.float32)
    r = rng.uniform(0.01, 0.08, 100000).astype(np.float32)
    exp = O.collides_many(t, c, r)
    got = P.collides_many(tree, torch.from_numpy(c).cuda(), torch.from_numpy(r).cuda())
    assert got.is_cuda and np.array_equal(got.cpu().numpy(), exp)
    words = P.query_bits(tree, torch.from_numpy(c).cuda(), torch.from_numpy(r).cuda())
    bits = np.unpackbits(words.cpu().numpy().view(np.uint8), bitorder="little")[:100000]
    assert np.array_equal(bits.astype(bool), exp)


def test_infinite_radius_with_infinite_centre():
    rng = np.random.default_rng(8)
    pts = rng.uniform(0, 1, (50, 3)).astype(np.float32)
    t = O.construct(pts, 0.01, 0.08)
    tree = upload(t)
    c = np.array([[np.inf, 0.5, 0.5], [np.nan, 0.5, 0.5], [0.5, 0.5, 0.5], [-np.inf, 0, 0]])
    r = np.array([np.inf, np.inf, np.inf, 0.05])
    for pre in (True, False):
        got = P.collides_many(tree, c, r, use_aabb_prefilter=pre, check_radii=False)
        assert np.array_equal(got, O.collides_many(t, c, r, use_aabb_prefilter=pre)), pre


@pytest.mark.parametrize("mode", ["thread", "warp", "hybrid"])
def test_unbinned_kernels(mode):
    """The unbinned kernels (one thread per sphere / one warp per sphere /
    thread classification + warp scans),
    forced through the C-ABI flags, against the oracle: float and float64
    inputs, non-finite and extreme values, every lane width, lane masks."""
    from paper_2406_02807_b200 import _lib
    from paper_2406_02807_b200 import workloads as W
    from paper_2406_02807_b200.query import _host_query
    flag = {"thread": _lib.MODE_THREAD, "warp": _lib.MODE_DIRECT | _lib.MODE_WARP,
            "hybrid": _lib.MODE_DIRECT}[mode]
    cloud = W.cfg1_cloud()
    t = O.construct(cloud, 0.02, 0.08)
    tree = upload(t)
    c, r = W.cfg1_queries(cloud, n_groups=1 << 12)
    exp = O.collides_many(t, c, r)
    for L in (1, 2, 8, 32):
        gb, _, _ = _host_query(tree, c, r, 0, L, None, True, True, mode=flag)
        assert np.array_equal(gb, exp.reshape(-1, L).any(1)), L
    rng = np.random.default_rng(5)
    m = rng.uniform(size=len(r)) < 0.7
    gb, _, _ = _host_query(tree, c, r, 0, 8, m, True, True, mode=flag)
    assert np.array_equal(gb, (exp & m).reshape(-1, 8).any(1))
    c64 = c.astype(np.float64) + rng.normal(0, 1e-9, c.shape)
    r64 = r.astype(np.float64)
    gb, _, _ = _host_query(tree, c64, r64, _lib.INPUT_F64, 1, None, True, True, mode=flag)
    assert np.array_equal(gb, O.collides_many(t, c64, r64))
    # non-finite / extreme spheres, with and without the AABB prefilter
    c2 = rng.uniform(-0.8, 0.8, (256, 3))
    c2[:, 2] = rng.uniform(0, 0.3, 256)
    r2 = rng.uniform(0.02, 0.08, 256)
    c2[0, 0], c2[1, 1], c2[2, 2], c2[3] = np.nan, np.inf, -np.inf, 1e30
    r2[4], r2[5], r2[6], r2[7], r2[8] = np.nan, 0.0, 1e30, -0.05, np.inf
    for pre in (True, False):
        gb, _, _ = _host_query(tree, c2, r2, _lib.INPUT_F64, 1, None, pre, False, mode=flag)
        assert np.array_equal(gb, O.collides_many(t, c2, r2, use_aabb_prefilter=pre)), pre
