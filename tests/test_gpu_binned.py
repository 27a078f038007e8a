"""Parity of the leaf-binned query pipeline (capt_binned.cu) with the oracle.

Every case forces CAPT_MODE_BINNED and, where useful, compares against the
direct kernel as well (both must equal the oracle bit for bit)."""

import numpy as np
import pytest

from conftest import golden_tree, load_golden
from oracle import oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2406_02807_b200")
from paper_2406_02807_b200 import _lib  # noqa: E402
from paper_2406_02807_b200 import workloads as W  # noqa: E402
from paper_2406_02807_b200.query import _host_inputs, _host_query  # noqa: E402

BINNED, DIRECT = _lib.MODE_BINNED, _lib.MODE_DIRECT
# the binned scan runs on the tensor cores by default; K5_FFMA selects the
# CUDA-core kernel -- both must give the reference's verdicts
K5 = {"tc": BINNED, "ffma": BINNED | _lib.K5_FFMA}


def upload(t):
    return P.Capt(t["k"], t["n_points"], t["r_min"], t["r_max"], t["tests"], t["aff_lo"],
                  t["aff_hi"], t["offsets"], t["aff_values"])


def q(tree, c, r, L=1, mask=None, prefilter=True, mode=BINNED):
    cc, rr, f64 = _host_inputs(tree, c, r)
    bits, _, bad = _host_query(tree, cc, rr, f64, L, mask, prefilter, False, mode=mode)
    return bits


@pytest.mark.parametrize("k5", ["tc", "ffma"])
def test_binned_golden_masks(k5):
    z = load_golden("queries.npz")
    for name in z["names"]:
        pts = z[f"{name}/points"]
        rmin, rmax = z[f"{name}/band"]
        tree = upload(O.construct(pts, rmin, rmax))
        c, r = z[f"{name}/centers"], z[f"{name}/radii"]
        n = len(r)
        exp = np.unpackbits(z[f"{name}/mask"])[:n].astype(bool)
        assert np.array_equal(q(tree, c, r, mode=K5[k5]), exp), name
        nopre = np.unpackbits(z[f"{name}/mask_nopre"])[:n].astype(bool)
        assert np.array_equal(q(tree, c, r, prefilter=False, mode=K5[k5]), nopre), name
        lane = np.unpackbits(z[f"{name}/lane_mask"])[:n].astype(bool)
        gb = np.unpackbits(z[f"{name}/group8"])[: n // 8].astype(bool)
        assert np.array_equal(q(tree, c, r, 8, lane.astype(np.uint8), mode=K5[k5]), gb), name


def test_binned_cfg0_golden():
    z = load_golden("cfg0.npz")
    tree = upload(golden_tree(z, ""))
    n = int(z["n_queries"][0])
    c, r = W.cfg0_queries()
    assert np.array_equal(q(tree, c[:n], r[:n]), np.unpackbits(z["mask"])[:n].astype(bool))
    # full config-0 batch: binned == direct == oracle
    exp = O.collides_many(golden_tree(z, ""), c, r)
    assert np.array_equal(q(tree, c, r), exp)
    assert np.array_equal(q(tree, c, r, mode=DIRECT), exp)


@pytest.mark.parametrize("L", [1, 2, 8, 32])
def test_binned_cfg1_groups(L):
    cloud = W.cfg1_cloud()
    t = O.construct(cloud, 0.02, 0.08)
    tree = upload(t)
    c, r = W.cfg1_queries(cloud, n_groups=1 << 16)
    per = O.collides_many(t, c, r)
    exp = per.reshape(-1, L).any(1)
    assert np.array_equal(q(tree, c, r, L), exp)
    if L == 8:
        assert np.array_equal(q(tree, c, r, 8, mode=DIRECT), exp)
        assert np.array_equal(O.collides_groups(t, c, r, 8), exp)


@pytest.mark.parametrize("k5", ["tc", "ffma"])
def test_binned_dense_gaussians_multichunk(k5):
    # dense mixture: affordance sets larger than one 1024-point shared-memory chunk
    cloud = W.cfg3_cloud(n=32768, n_comp=8, seed=5)
    t = O.construct(cloud, 0.01, 0.1)
    assert np.diff(t["offsets"]).max() > 1024
    tree = upload(t)
    c, r = W.cfg3_queries(1 << 19, seed=7)
    exp = O.collides_many(t, c, r)
    assert np.array_equal(q(tree, c, r, mode=K5[k5]), exp)


def test_binned_f64_and_nonfinite():
    rng = np.random.default_rng(17)
    pts = rng.uniform(0, 1, (3000, 3)).astype(np.float32)
    t = O.construct(pts, 0.01, 0.08)
    tree = upload(t)
    c = rng.uniform(-0.1, 1.1, (300000, 3))
    r = rng.uniform(0.01, 0.08, 300000)
    c[:1000] = c[:1000].astype(np.float32)  # some fp32-exact rows
    r[:1000] = r[:1000].astype(np.float32)
    c[5, 0] = np.nan
    c[6, 1] = np.inf
    r[7] = np.nan
    exp = O.collides_many(t, c, r)
    assert np.array_equal(q(tree, c, r), exp)


@pytest.mark.parametrize("k5", ["tc", "ffma"])
def test_binned_tangency_heavy(k5):
    # spheres exactly tangent (in float64) to cloud points: exercises the
    # ambiguous-band rescan inside the binned kernel
    rng = np.random.default_rng(23)
    pts = rng.uniform(0, 1, (4096, 3)).astype(np.float32)
    t = O.construct(pts, 0.01, 0.08)
    tree = upload(t)
    n = 1 << 18
    idx = rng.integers(0, len(pts), n)
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    r = W.clamp_radii(rng.uniform(0.01, 0.08, n).astype(np.float32), 0.01, 0.08)
    c = (pts[idx].astype(np.float64) + d * r[:, None].astype(np.float64)).astype(np.float32)
    exp = O.collides_many(t, c, r)
    got = q(tree, c, r, mode=K5[k5])
    assert np.array_equal(got, exp)
    assert np.array_equal(got, O.brute_collides_many(pts, c, r))


def test_binned_device_built_tree_and_auto_mode():
    cloud = W.cfg1_cloud()
    tree = P.construct(P.PointCloud(cloud), P.BuildParams(0.02, 0.08))
    c, r = W.cfg1_queries(cloud, n_groups=1 << 15, seed=3)
    exp = O.brute_collides_many(cloud, c, r)
    assert np.array_equal(P.collides_many(tree, c, r), exp)  # auto -> hybrid here
    assert np.array_equal(q(tree, c, r, mode=DIRECT), exp)
    assert np.array_equal(q(tree, c, r), exp)  # forced binned
    c2, r2 = W.cfg1_queries(cloud, n_groups=1 << 18, seed=4)  # 2 M spheres: auto -> binned
    assert np.array_equal(P.collides_many(tree, c2, r2), O.collides_many(O.tree_from(tree), c2, r2))


def test_binned_split_walls_and_grid_cells():
    # lattice cloud: many split values shared by queries that sit exactly on
    # split walls (x == T goes left) and on descent-grid cell boundaries
    ax = np.linspace(-1, 1, 24, dtype=np.float32)
    pts = np.stack(np.meshgrid(ax, ax, ax, indexing="ij"), -1).reshape(-1, 3)
    t = O.construct(pts, 0.01, 0.12)
    tree = upload(t)
    rng = np.random.default_rng(9)
    n = 1 << 18
    c = pts[rng.integers(0, len(pts), n)].copy()
    jitter = rng.integers(0, 3, (n, 3)).astype(np.float32) * np.float32(ax[1] - ax[0]) / 2
    c = (c + jitter).astype(np.float32)
    r = W.clamp_radii(rng.uniform(0.01, 0.12, n).astype(np.float32), 0.01, 0.12)
    assert np.array_equal(P.leaf_indices(tree, c), O.leaf_indices(t, c))
    exp = O.collides_many(t, c, r)
    assert np.array_equal(q(tree, c, r), exp)
    assert np.array_equal(q(tree, c, r, mode=DIRECT), exp)


def test_host_pipeline_chunks_counters_and_bad_radius():
    # host buffers larger than one pipeline chunk (4M spheres): two-stream
    # chunked path; verdict words, counters and the first bad index must all
    # match the single-shot device path / the oracle
    cloud = W.cfg1_cloud()
    t = O.construct(cloud, 0.02, 0.08)
    tree = upload(t)
    c, r = W.cfg1_queries(cloud, n_groups=(1 << 20) + 96, seed=77)  # 8.4M spheres, 3 chunks
    exp = O.collides_groups(t, c, r, 8)
    bits, cnt, _ = _host_query(tree, c, r, 0, 8, None, True, True, stats=True)
    assert np.array_equal(bits, exp)
    e_hits, e_rej, e_scanned = O.collides_groups(t, c, r, 8, return_counters=True)[1]
    assert int(cnt[0]) == e_hits and int(cnt[4]) == e_rej and int(cnt[2]) == e_scanned
    bits2, _, _ = _host_query(tree, c, r, 0, 8, None, True, True)
    assert np.array_equal(bits2, exp)
    r_bad = r.copy()
    r_bad[5_000_001] = 0.5
    r_bad[7_000_000] = 0.001
    with pytest.raises(ValueError, match="radius 0.5 outside"):
        P.collides_many(tree, c, r_bad)


@pytest.mark.parametrize("k5", ["tc", "ffma"])
def test_binned_aabb_boundary_spheres(k5):
    """Spheres whose centre lies exactly r (and one ulp either side) outside a
    leaf's affordance box: the binned path's conservative fp32 AABB filter
    must give the reference verdict (the reference's own float64 AABB test is
    never the deciding factor, but these are the cases that stress it)."""
    rng = np.random.default_rng(77)
    pts = rng.uniform(0, 1, (3000, 3)).astype(np.float32)
    t = O.construct(pts, 0.01, 0.08)
    tree = upload(t)
    lo, hi = t["aff_lo"].reshape(-1, 3), t["aff_hi"].reshape(-1, 3)
    leaves = rng.integers(0, len(lo), 4000)
    ok = np.isfinite(lo).all(1) & np.isfinite(hi).all(1)  # empty sets have +inf boxes
    leaves = leaves[ok[leaves]]
    r = rng.uniform(0.01, 0.08, len(leaves)).astype(np.float32)
    ax = rng.integers(0, 3, len(leaves))
    c = rng.uniform(lo[leaves], hi[leaves]).astype(np.float32)
    side = rng.integers(0, 2, len(leaves)).astype(bool)
    idx = np.arange(len(leaves))
    c[idx, ax] = np.where(side, hi[leaves, ax] + r, lo[leaves, ax] - r)
    cs = [c]
    for d in (-1, 1):  # one ulp inward / outward
        c2 = c.copy()
        c2[idx, ax] = np.nextafter(c[idx, ax], c[idx, ax] + d * np.float32(1.0))
        cs.append(c2)
    c = np.concatenate(cs)
    r = np.concatenate([r] * 3)
    exp = O.collides_many(t, c, r)
    assert np.array_equal(q(tree, c, r, mode=K5[k5]), exp)
    assert np.array_equal(q(tree, c, r, mode=DIRECT), exp)
    n8 = len(r) // 8 * 8
    assert np.array_equal(q(tree, c[:n8], r[:n8], 8, mode=K5[k5]),
                          exp[:n8].reshape(-1, 8).any(1))


def test_binned_many_leaves_device_scans():
    # > 32768 leaves: per-leaf starts and tile indices come from device-wide
    # scans instead of the one-CTA pass
    rng = np.random.default_rng(41)
    pts = rng.uniform(0, 1, (40000, 3)).astype(np.float32)
    t = O.construct(pts, 0.005, 0.03)
    assert t["n"] > 32768
    tree = upload(t)
    c = rng.uniform(0, 1, (1 << 20, 3)).astype(np.float32)
    r = rng.uniform(0.005, 0.03, 1 << 20).astype(np.float32)
    exp = O.collides_many(t, c, r)
    for k5 in ("tc", "ffma"):
        assert np.array_equal(q(tree, c, r, mode=K5[k5]), exp), k5
