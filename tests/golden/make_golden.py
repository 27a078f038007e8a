"""Generate golden fixtures by running the REAL reference package.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``captree`` read-only from /root/reference/pkg/src and records its
outputs on seeded inputs as small .npz files next to this script.  The GPU box
never needs the reference: the tests read only these fixtures.  Inputs are
regenerated from the seeds stored in each fixture, and also stored directly
when small.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import captree  # noqa: E402  (the reference)
from captree import (BuildParams, FilterConfig, PointCloud, Sphere, SphereBatch,  # noqa: E402
                     collides_batch, collides_many, construct, filter_cloud)
from captree.geom import Aabb  # noqa: E402
from captree.morton import morton_keys  # noqa: E402
from captree.tree import leaf_indices  # noqa: E402

from oracle import oracle as O  # noqa: E402  (canonical ordering helper only)
from paper_2406_02807_b200 import workloads as W  # noqa: E402


def tree_arrays(tree, prefix):
    return {
        f"{prefix}tests": tree.tests, f"{prefix}aff_lo": tree.aff_lo,
        f"{prefix}aff_hi": tree.aff_hi, f"{prefix}offsets": tree.offsets,
        f"{prefix}canon": O.canonical_values(tree),
        f"{prefix}meta": np.array([tree.k, tree.n, tree.n_points], np.int64),
        f"{prefix}band": np.array([tree.r_min, tree.r_max], np.float64),
    }


def tangency(rng, pts, count, r_lo, r_hi):
    p = pts.astype(np.float64)
    idx = rng.integers(0, len(p), size=count)
    r = rng.uniform(r_lo, r_hi, size=count)
    d = rng.normal(size=(count, p.shape[1]))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return p[idx] + d * r[:, None], r


def make_trees():
    """Trees over assorted clouds: padding, duplicates, shortcut on/off, k=2."""
    out = {}
    cases = []
    rng = np.random.default_rng(1234)
    for n in (1, 2, 3, 5, 100, 200, 777, 1024):
        cases.append((f"u{n}", rng.uniform(0, 1, (n, 3)).astype(np.float32), 0.01, 0.08, True))
    cases.append(("u777_nosc", rng.uniform(0, 1, (777, 3)).astype(np.float32), 0.01, 0.08, False))
    dup = rng.uniform(0, 1, (300, 3)).astype(np.float32)
    cases.append(("dup900", np.repeat(dup, 3, axis=0), 0.01, 0.08, True))
    cases.append(("dense256", rng.uniform(0, 0.004, (256, 3)).astype(np.float32), 0.01, 0.08, True))
    cases.append(("dense256_nosc", rng.uniform(0, 0.004, (256, 3)).astype(np.float32), 0.01, 0.08, False))
    cases.append(("k2_64", rng.uniform(0, 1, (64, 2)).astype(np.float32), 0.01, 0.08, True))
    cases.append(("wide_band", rng.uniform(-1, 1, (500, 3)).astype(np.float32), 0.05, 0.3, True))
    cases.append(("cfg1_1k", W.cfg1_cloud(1024, seed=7), 0.02, 0.08, True))
    names = []
    for name, pts, rmin, rmax, sc in cases:
        tree = construct(PointCloud(pts), BuildParams(rmin, rmax), use_rmin_shortcut=sc)
        out.update(tree_arrays(tree, f"{name}/"))
        out[f"{name}/points"] = pts
        out[f"{name}/shortcut"] = np.array([int(sc)])
        names.append(name)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "trees.npz"), **out)
    print("trees.npz", len(names), "trees")


def make_queries():
    """Masks from collides_many (prefilter on/off), leaf indices, and group bits
    from collides_batch, on fp32 inputs incl. tangency spheres and exact band
    edges (test_acceptance.py:54-91 pattern)."""
    out = {}
    rng = np.random.default_rng(4321)
    specs = [
        ("u300", rng.uniform(0, 1, (300, 3)).astype(np.float32), 0.01, 0.08),
        ("u100pad", rng.uniform(0, 1, (100, 3)).astype(np.float32), 0.01, 0.08),
        ("dup600", np.repeat(rng.uniform(0, 1, (200, 3)).astype(np.float32), 3, 0), 0.01, 0.08),
        ("cfg1_2k", W.cfg1_cloud(2048, seed=9), 0.02, 0.08),
        ("k2_200", rng.uniform(0, 1, (200, 2)).astype(np.float32), 0.01, 0.08),
    ]
    names = []
    for name, pts, rmin, rmax in specs:
        k = pts.shape[1]
        tree = construct(PointCloud(pts), BuildParams(rmin, rmax))
        lo = pts.min(0).astype(np.float64) - 2 * rmax
        hi = pts.max(0).astype(np.float64) + 2 * rmax
        c1 = rng.uniform(lo, hi, size=(6000, k))
        r1 = rng.uniform(rmin, rmax, size=6000)
        c2, r2 = tangency(rng, pts, 2000, rmin, rmax)
        c = np.concatenate([c1, c2]).astype(np.float32)
        r = np.concatenate([r1, r2]).astype(np.float32)
        r = W.clamp_radii(r, rmin, rmax)
        r[0], r[1] = W.f32_band(rmin, rmax)
        c64, r64 = c.astype(np.float64), r.astype(np.float64)
        out[f"{name}/points"] = pts
        out[f"{name}/band"] = np.array([rmin, rmax])
        out[f"{name}/centers"] = c
        out[f"{name}/radii"] = r
        out[f"{name}/mask"] = np.packbits(collides_many(tree, c64, r64))
        out[f"{name}/mask_nopre"] = np.packbits(
            collides_many(tree, c64, r64, use_aabb_prefilter=False))
        out[f"{name}/leaf"] = leaf_indices(tree, c64).astype(np.int32)
        # groups of 8 with a random validity mask
        L = 8
        lane_mask = rng.uniform(size=len(r)) < 0.8
        gbits = []
        scanned = []
        for g in range(len(r) // L):
            s = slice(g * L, (g + 1) * L)
            o = collides_batch(tree, SphereBatch(c64[s], r64[s], lane_mask[s]),
                               collect_stats=True)
            gbits.append(o.any_collision)
            scanned.append(o.points_scanned)
        out[f"{name}/lane_mask"] = np.packbits(lane_mask)
        out[f"{name}/group8"] = np.packbits(np.array(gbits))
        out[f"{name}/group8_scanned"] = np.array(scanned, np.int64)
        names.append(name)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "queries.npz"), **out)
    print("queries.npz", len(names), "clouds")


def make_hand_cases():
    """Known answers from the reference's own tests (test_query.py:18-23,
    172-179; test_tree.py:27-57; test_morton.py:13-19,44-49)."""
    out = {}
    pts = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], np.float32)
    tree = construct(PointCloud(pts), BuildParams(0.01, 2.0))
    cs = np.array([[0.0, 0.0, 0.05], [0.5, 0.5, 0.5], [2.0, 0.0, 0.0],
                   [1.5, 0.0, 0.0], [1.5, 0.0, 0.0], [1.5, 0.0, 0.0]])
    rs = np.array([0.1, 0.5, 1.0, 0.5, np.nextafter(0.5, 0.0), np.nextafter(0.5, 1.0)])
    out["tiny/points"] = pts
    out["tiny/centers"] = cs
    out["tiny/radii"] = rs
    out["tiny/expect"] = collides_many(tree, cs, rs)
    out.update(tree_arrays(tree, "tiny/"))
    # morton known answers
    b = Aabb(np.array([0.0, -1.0, 2.0]), np.array([1.0, 1.0, 5.0]))
    out["morton/lo_hi_keys"] = morton_keys(np.stack([b.lo, b.hi]), b, (0, 1, 2))
    b2 = Aabb(np.zeros(3), np.ones(3))
    q = np.array([[0, 0, 0], [0, 0, 1], [0, 1, 0], [1, 0, 0], [0.25, 0.75, 0.5]], np.float64)
    perms = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]
    out["morton/unit_pts"] = q
    out["morton/unit_keys"] = np.stack([morton_keys(q, b2, p) for p in perms])
    rng = np.random.default_rng(99)
    rp = rng.uniform(-1, 1, (64, 3)).astype(np.float32)
    rb = Aabb(rp.min(0).astype(np.float64), rp.max(0).astype(np.float64))
    out["morton/rand_pts"] = rp
    out["morton/rand_keys"] = np.stack([morton_keys(rp, rb, p) for p in perms])
    np.savez_compressed(os.path.join(HERE, "hand.npz"), **out)
    print("hand.npz")


def make_filters():
    """filter_cloud outputs (test_oracle.py:97-120 grid, plus reach, k=2,
    duplicates, and a 20k-point slice of the config-2 depth cloud)."""
    out = {}
    rng = np.random.default_rng(61)
    names = []
    for n in (1, 2, 17, 300, 1500):
        pts = rng.uniform(0, 1, (n, 3)).astype(np.float32)
        for r in (0.0, 0.02, 0.07, 0.2):
            name = f"u{n}_r{r}"
            out[f"{name}/points"] = pts
            out[f"{name}/r"] = np.array([r])
            out[f"{name}/out"] = filter_cloud(PointCloud(pts), FilterConfig(r)).points
            names.append(name)
    pts = rng.uniform(-1, 1, (800, 3)).astype(np.float32)
    base = np.array([0.2, 0.0, -0.1])
    out["reach/points"] = pts
    out["reach/r"] = np.array([0.05])
    out["reach/base"] = base
    out["reach/max_reach"] = np.array([0.8])
    out["reach/out"] = filter_cloud(PointCloud(pts), FilterConfig(0.05, base=base, max_reach=0.8)).points
    names.append("reach")
    k2 = rng.uniform(0, 1, (700, 2)).astype(np.float32)
    out["k2/points"] = k2
    out["k2/r"] = np.array([0.03])
    out["k2/out"] = filter_cloud(PointCloud(k2), FilterConfig(0.03)).points
    names.append("k2")
    dup = np.repeat(rng.uniform(0, 1, (400, 3)).astype(np.float32), 3, 0)
    out["dup/points"] = dup
    out["dup/r"] = np.array([0.01])
    out["dup/out"] = filter_cloud(PointCloud(dup), FilterConfig(0.01)).points
    names.append("dup")
    raw = W.cfg2_raw_cloud()
    sl = raw[rng.choice(len(raw), 20000, replace=False)]
    out["cfg2_20k/points"] = sl
    out["cfg2_20k/r"] = np.array([0.01])
    out["cfg2_20k/out"] = filter_cloud(PointCloud(sl), FilterConfig(0.01)).points
    names.append("cfg2_20k")
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "filters.npz"), **out)
    print("filters.npz", len(names))


def make_cfg0_slice():
    """Config 0 (the reference's own CPU-runnable case): the full tree and the
    reference masks of the first 131072 queries."""
    pts = W.cfg0_cloud()
    tree = construct(PointCloud(pts), BuildParams(0.01, 0.08))
    c, r = W.cfg0_queries()
    n = 131072
    out = tree_arrays(tree, "")
    out["n_queries"] = np.array([n])
    out["mask"] = np.packbits(collides_many(tree, c[:n].astype(np.float64),
                                            r[:n].astype(np.float64)))
    out["centers_sha"] = np.frombuffer(__import__("hashlib").sha1(c[:n].tobytes()).digest(), np.uint8)
    np.savez_compressed(os.path.join(HERE, "cfg0.npz"), **out)
    print("cfg0.npz")



def make_trace():
    """A mixed trace from the reference's own generator (synth.gen_queries),
    written by its writer, and the reference's replay verdicts
    (bench.capt_verdicts) on the tree over the same cloud."""
    from captree.bench import capt_verdicts
    from captree.io import read_trace, write_trace
    from captree.synth import gen_queries
    rng = np.random.default_rng(77)
    pts = rng.uniform(-1, 1, (3000, 3)).astype(np.float32)
    cloud = PointCloud(pts)
    params = BuildParams(0.02, 0.08)
    tree = construct(cloud, params)
    out = {"points": pts, "band": np.array([0.02, 0.08])}
    for name, batch in (("b8", 8), ("b5", 5), ("b40", 40)):
        recs = gen_queries(cloud, params, 2000, workload="mixed", batch_size=batch, seed=batch)
        path = os.path.join("/tmp", f"capt_trace_{name}.csv")
        write_trace(recs, path)
        with open(path, "rb") as f:
            out[f"{name}/csv"] = np.frombuffer(f.read(), np.uint8)
        back = read_trace(path)
        out[f"{name}/verdicts"] = capt_verdicts(tree, back)
        out[f"{name}/nopre"] = capt_verdicts(tree, back, use_aabb_prefilter=False)
        out[f"{name}/batch_ids"] = np.array([r.batch_id for r in back], np.int64)
        out[f"{name}/sizes"] = np.array([len(r) for r in back], np.int64)
        out[f"{name}/expected"] = np.array([-1 if r.expected is None else int(r.expected)
                                            for r in back], np.int64)
        os.remove(path)
    np.savez_compressed(os.path.join(HERE, "trace.npz"), **out)


def make_dispersion():
    """dispersion_stats (oracle.py:141-158) on assorted clouds, plus the
    per-point values of the float64 cKDTree query it is built on."""
    from scipy import __version__ as scipy_version
    from scipy.spatial import cKDTree
    from captree.oracle import dispersion_stats
    rng = np.random.default_rng(91)
    clouds = {
        "uniform": rng.uniform(-1, 1, (5000, 3)).astype(np.float32),
        "dups": np.repeat(rng.uniform(0, 1, (700, 3)).astype(np.float32), 3, axis=0),
        "k2": rng.normal(0, 0.1, (3000, 2)).astype(np.float32),
        "cfg1": W.cfg1_cloud(),
        "tiny": np.array([[0, 0, 0], [1, 0, 0]], np.float32),
    }
    out = {"scipy": np.frombuffer(scipy_version.encode(), np.uint8)}
    for name, pts in clouds.items():
        st = dispersion_stats(PointCloud(pts))
        p64 = pts.astype(np.float64)
        nn = cKDTree(p64).query(p64, k=2)[0][:, 1]
        out[f"{name}/points"] = pts
        out[f"{name}/stats"] = np.array([st.mean, st.median, st.p95, st.count], np.float64)
        out[f"{name}/nn"] = nn
    np.savez_compressed(os.path.join(HERE, "dispersion.npz"), **out)


def make_capt_files():
    """.capt dumps written by the reference's own save_capt (tree.py:276-288):
    a 3-D tree with padding leaves, the r_min shortcut and duplicates, and a
    k = 2 tree, plus queries and the reference's masks on the loaded trees."""
    from captree.tree import load_capt, save_capt
    rng = np.random.default_rng(4321)
    pts3 = np.concatenate([rng.uniform(-1, 1, (700, 3)),
                           np.repeat(rng.uniform(0, 0.2, (20, 3)), 3, axis=0)]).astype(np.float32)
    pts2 = rng.normal(0, 0.3, (300, 2)).astype(np.float32)
    out = {}
    for name, pts, band in (("ref3d", pts3, (0.02, 0.15)), ("ref2d", pts2, (0.01, 0.1))):
        tree = construct(PointCloud(pts), BuildParams(*band))
        path = os.path.join(HERE, f"{name}.capt")
        save_capt(tree, path)
        back = load_capt(path)  # (r_min / r_max come back as fp32 values)
        k = pts.shape[1]
        c = rng.uniform(pts.min(0) - 0.2, pts.max(0) + 0.2, (4096, k))
        r = rng.uniform(back.r_min, back.r_max, 4096)
        r = np.clip(r, np.nextafter(np.float32(back.r_min), np.float32(1)), back.r_max)
        out[f"{name}/centers"] = c
        out[f"{name}/radii"] = r
        out[f"{name}/mask"] = np.packbits(collides_many(back, c, r))
    np.savez_compressed(os.path.join(HERE, "capt_files.npz"), **out)


if __name__ == "__main__":
    print("reference", captree.__version__, "numpy", np.__version__)
    if len(sys.argv) > 1:  # regenerate only the named fixtures, e.g. capt_files
        for name in sys.argv[1:]:
            globals()[f"make_{name}"]()
        sys.exit(0)
    make_hand_cases()
    make_trees()
    make_queries()
    make_filters()
    make_cfg0_slice()
    make_trace()
    make_dispersion()
    make_capt_files()
