"""Pin the CPU oracle (oracle/) against fixtures produced by the real
reference (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import golden_tree, load_golden
from oracle import oracle as O


def _same_tree(a, b):
    """Bit-exact Capt arrays; per-leaf sets compared in canonical order.  With
    straddling ties at a split (a["ties"] > 0) leaf membership depends on
    np.argpartition's permutation, so only T and the set sizes and
    boxes are compared."""
    assert np.array_equal(a["tests"], b["tests"])
    assert np.array_equal(a["offsets"], b["offsets"])
    assert np.array_equal(a["aff_lo"], b["aff_lo"])
    assert np.array_equal(a["aff_hi"], b["aff_hi"])
    if a.get("ties", 0) == 0:
        assert np.array_equal(O.canonical_values(a), O.canonical_values(b))


def test_oracle_trees_match_reference():
    z = load_golden("trees.npz")
    for name in z["names"]:
        ref = golden_tree(z, f"{name}/")
        mine = O.construct(z[f"{name}/points"], ref["r_min"], ref["r_max"],
                           bool(z[f"{name}/shortcut"][0]))
        assert mine["ties"] == 0 or name.startswith("dup"), name
        _same_tree(mine, ref)


def test_oracle_queries_match_reference():
    z = load_golden("queries.npz")
    for name in z["names"]:
        pts = z[f"{name}/points"]
        rmin, rmax = z[f"{name}/band"]
        tree = O.construct(pts, rmin, rmax)
        c = z[f"{name}/centers"].astype(np.float64)
        r = z[f"{name}/radii"].astype(np.float64)
        n = len(r)
        mask = np.unpackbits(z[f"{name}/mask"])[:n].astype(bool)
        nopre = np.unpackbits(z[f"{name}/mask_nopre"])[:n].astype(bool)
        assert np.array_equal(O.collides_many(tree, c, r), mask), name
        assert np.array_equal(O.collides_many(tree, c, r, use_aabb_prefilter=False), nopre), name
        assert np.array_equal(O.leaf_indices(tree, c), z[f"{name}/leaf"]), name
        lane = np.unpackbits(z[f"{name}/lane_mask"])[:n].astype(bool)
        g, cnt = O.collides_groups(tree, c, r, 8, mask=lane, return_counters=True)
        gb = np.unpackbits(z[f"{name}/group8"])[: n // 8].astype(bool)
        assert np.array_equal(g, gb), name
        assert cnt[2] == int(z[f"{name}/group8_scanned"].sum()), name
        # brute force agrees with the tree (oracle.py:34-49)
        assert np.array_equal(O.brute_collides_many(pts, c, r), mask), name


def test_oracle_hand_cases():
    z = load_golden("hand.npz")
    tree = O.construct(z["tiny/points"], 0.01, 2.0)
    _same_tree(tree, golden_tree(z, "tiny/"))
    got = O.collides_many(tree, z["tiny/centers"], z["tiny/radii"])
    assert np.array_equal(got, z["tiny/expect"])
    assert list(got) == [True, False, True, True, False, True]


def test_oracle_morton_keys():
    z = load_golden("hand.npz")
    keys = O.morton_keys(np.array([[0, -1, 2], [1, 1, 5]], np.float32),
                         [0.0, -1.0, 2.0], [1.0, 1.0, 5.0], (0, 1, 2))
    assert list(keys) == [0, (1 << 63) - 1]
    assert np.array_equal(keys, z["morton/lo_hi_keys"])
    perms = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]
    for i, p in enumerate(perms):
        got = O.morton_keys(z["morton/unit_pts"].astype(np.float32), np.zeros(3), np.ones(3), p)
        assert np.array_equal(got, z["morton/unit_keys"][i])
        rp = z["morton/rand_pts"]
        got = O.morton_keys(rp, rp.min(0).astype(np.float64), rp.max(0).astype(np.float64), p)
        assert np.array_equal(got, z["morton/rand_keys"][i])


def test_oracle_filter_matches_reference():
    z = load_golden("filters.npz")
    for name in z["names"]:
        pts = z[f"{name}/points"]
        r = float(z[f"{name}/r"][0])
        if f"{name}/base" in z:
            got = O.filter_cloud(pts, r, base=z[f"{name}/base"],
                                 max_reach=float(z[f"{name}/max_reach"][0]))
        else:
            got = O.filter_cloud(pts, r)
        assert np.array_equal(got, z[f"{name}/out"]), name


def test_oracle_cfg0_slice():
    from paper_2406_02807_b200 import workloads as W
    z = load_golden("cfg0.npz")
    tree = O.construct(W.cfg0_cloud(), 0.01, 0.08)
    _same_tree(tree, golden_tree(z, ""))
    n = int(z["n_queries"][0])
    c, r = W.cfg0_queries()
    import hashlib
    assert hashlib.sha1(c[:n].tobytes()).digest() == bytes(z["centers_sha"])
    got = O.collides_many(tree, c[:n].astype(np.float64), r[:n].astype(np.float64))
    assert np.array_equal(got, np.unpackbits(z["mask"])[:n].astype(bool))
