"""Full-size parity at the benchmarked configurations (BASELINE.json configs
1-3): the device tree equals the oracle's construct of the same cloud (T,
offsets, boxes bit for bit, every affordance set in canonical order), the
device filter equals the oracle's filter_cloud, and EVERY verdict of the
benchmarked batch -- through the default (auto) pipeline, device-resident
inputs, as bench.py times it -- equals the oracle's collides_many /
collides_batch (query.py:184-219, 126-167).  The oracle runs on every host
thread; the whole file takes a minute or two."""

import numpy as np
import pytest

from oracle import oracle as O
from oracle.parity import mask_parity, tree_parity

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2406_02807_b200")
torch = pytest.importorskip("torch")
from paper_2406_02807_b200 import workloads as W  # noqa: E402


def device_words(tree, c, r, L):
    cd, rd = torch.from_numpy(c).cuda(), torch.from_numpy(r).cuda()
    bad = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    w = P.query_bits(tree, cd, rd, L, first_bad=bad, check_radii=True)
    torch.cuda.synchronize()
    assert int(bad.item()) == -1
    return w.cpu().numpy()


def check_tree(tree, cloud, r_min, r_max):
    tp = tree_parity(tree, cloud, r_min, r_max)
    ref = tp.pop("ref")
    assert tp["mismatches"] == 0, tp
    return ref


def test_cfg1_full_batch():
    cloud = W.cfg1_cloud()
    tree = P.construct(P.PointCloud(cloud), P.BuildParams(0.02, 0.08))
    ref = check_tree(tree, cloud, 0.02, 0.08)
    c, r = W.cfg1_queries(cloud)  # 4,194,304 groups x 8 spheres
    m = mask_parity(ref, c, r, device_words(tree, c, r, 8), 8, boundary=False)
    assert m["units"] == 4 << 20 and m["mismatches"] == 0, m


def test_cfg2_full_pipeline():
    raw = W.cfg2_raw_cloud()
    filt = P.filter_cloud(P.PointCloud(raw), P.FilterConfig(0.01)).points
    exp = O.filter_cloud(raw, 0.01)
    assert filt.shape == exp.shape
    assert np.array_equal(filt.view(np.uint32), exp.view(np.uint32))
    tree = P.construct(P.PointCloud(filt), P.BuildParams(0.01, 0.08))
    ref = check_tree(tree, filt, 0.01, 0.08)
    c, r = W.cfg2_queries(filt)  # 16,777,216 spheres
    m = mask_parity(ref, c, r, device_words(tree, c, r, 1), 1)
    assert m["spheres"] == 16 << 20 and m["mismatches"] == 0, m


def test_cfg3_full_tree_and_batch():
    cloud = W.cfg3_cloud()
    tree = P.construct(P.PointCloud(cloud), P.BuildParams(0.01, 0.1))
    ref = check_tree(tree, cloud, 0.01, 0.1)  # all 262,144 leaves, 475 M rows
    c, r = W.cfg3_queries()  # 67,108,864 spheres
    m = mask_parity(ref, c, r, device_words(tree, c, r, 1), 1)
    assert m["spheres"] == 64 << 20 and m["mismatches"] == 0, m
