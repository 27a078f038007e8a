"""The clearance-field query pipeline (csrc/capt_field.cu) against the oracle.

The field resolves most in-band spheres from a per-cell witness point and a
certified nearest-point lower bound (K0), then from the cell's candidate list
(its nearest cloud points and a bound on every other point); everything else
goes through the tree path.  Every case forces CAPT_MODE_FIELD and must equal
the oracle's collides_many / group bits (query.py:184-219, 126-167) bit for
bit; the field records themselves are checked against float64
nearest-neighbour distances."""

import numpy as np
import pytest

from conftest import golden_tree, load_golden
from oracle import oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2406_02807_b200")
from paper_2406_02807_b200 import _lib  # noqa: E402
from paper_2406_02807_b200 import workloads as W  # noqa: E402
from paper_2406_02807_b200.query import _host_inputs, _host_query  # noqa: E402

FIELD = _lib.MODE_FIELD


def upload(t):
    return P.Capt(t["k"], t["n_points"], t["r_min"], t["r_max"], t["tests"], t["aff_lo"],
                  t["aff_hi"], t["offsets"], t["aff_values"])


def q(tree, c, r, L=1, mask=None, prefilter=True, check=False, mode=FIELD):
    cc, rr, f64 = _host_inputs(tree, c, r)
    bits, _, bad = _host_query(tree, cc, rr, f64, L, mask, prefilter, check, mode=mode)
    return bits if not check else (bits, bad)


def centres(f):
    nz, ny, nx = f["shape"]
    c0, h = f["c0"].astype(np.float64), np.float64(f["h"])
    # fma(i, h, c0) rounded to fp32 (the product is exact in fp64)
    ax = [np.float32(np.arange(n, dtype=np.float64) * h + c0[d])
          for d, n in enumerate((nx, ny, nz))]
    return ax


def check_field(tree, cloud, sample=200000, seed=0):
    from scipy.spatial import cKDTree
    f = tree.clearance_field(cells=True, candidates=True)
    assert f is not None
    cells = f["cells"].reshape(-1, 8)
    K = f["n_cand"]
    cand = f["candidates"].reshape(-1, K, 3)
    nz, ny, nx = f["shape"]
    assert f["n_cells"] == nx * ny * nz <= int((1 << 21) * 1.05)
    pts = np.unique(cloud.astype(np.float32), axis=0).astype(np.float64)
    assert np.array_equal(f["box_lo"], cloud.min(0)) and np.array_equal(f["box_hi"], cloud.max(0))
    ax = centres(f)
    rng = np.random.default_rng(seed)
    idx = np.arange(len(cells)) if len(cells) <= sample else rng.choice(len(cells), sample, False)
    iz, rem = np.divmod(idx, ny * nx)
    iy, ix = np.divmod(rem, nx)
    x0 = np.stack([ax[0][ix], ax[1][iy], ax[2][iz]], 1).astype(np.float64)
    kt = cKDTree(cloud.astype(np.float64))  # (duplicates kept: they are distinct candidates)
    dk, _ = kt.query(x0, k=K + 1)
    nn = dk[:, 0]
    rec = cells[idx].astype(np.float64)
    rcap = np.float64(f["rcap"])
    # rec[3]: a certified lower bound of the 2nd-nearest distance (one fp32
    # ulp of slack for the centre's double rounding here), tight inside rcap
    slack = 2.0 * np.spacing(np.abs(x0).max(1).astype(np.float32)).astype(np.float64)
    assert np.all(rec[:, 3] <= dk[:, 1] + slack)
    assert np.all(rec[:, 3] <= rcap)
    in2 = dk[:, 1] < rcap * (1 - 1e-6)
    assert np.allclose(rec[in2, 3], dk[in2, 1], rtol=1e-5, atol=1e-7)
    # the witness: the nearest cloud point (+inf when none lies within rcap)
    has = np.isfinite(rec[:, 0])
    assert np.all(nn[~has] > rcap * (1 - 1e-6))
    near = nn < rcap * (1 - 1e-6)
    assert np.all(has[near])
    # (beyond rcap the witness is only the nearest point of the 27 buckets)
    dw = np.linalg.norm(x0[near] - rec[near, :3], axis=1)
    assert np.allclose(dw, nn[near], rtol=1e-5, atol=1e-7)
    wset = {tuple(p) for p in cloud.astype(np.float32)[:, :3].tolist()}
    assert all(tuple(w) in wset for w in rec[has][:2000, :3].astype(np.float32).tolist())
    # rec[6]: the second record's bound -- the distance of the first point
    # after its rec[7] candidates (the 2nd .. nearest), a multiple of q_step,
    # tight to one step inside rcap
    k2 = int(rec[0, 7])
    assert k2 in (2, 5) and np.all(rec[:, 7] == k2)
    assert np.all(rec[:, 6] <= dk[:, k2 + 1] + slack) and np.all(rec[:, 6] <= rcap)
    t2 = dk[:, k2 + 1] < rcap * (1 - 1e-3)
    assert np.all(rec[t2, 6] >= dk[t2, k2 + 1] - 2 * np.float64(f["q_step"]) - 1e-6 * rcap)
    # candidate records: the K nearest cloud points of x0 as int16 offsets
    # (distances equal to the float64 K-nearest distances within the offset
    # rounding where those lie inside rcap), and kd a lower bound of the
    # (K+1)-th nearest distance, tight (to one step) inside rcap
    step = np.float64(f["q_step"])
    assert step == 2.0 ** np.round(np.log2(step)) and 32767 * step >= rcap
    assert f["q_err"] >= np.sqrt(3) * step / 2
    kd = rec[:, 4]
    assert np.all(kd <= dk[:, K] + slack) and np.all(kd <= rcap)
    cnt = rec[:, 5].astype(int)
    off = cand[idx].astype(np.float64)
    fin = np.isfinite(off[:, :, 0])
    assert np.array_equal(fin.sum(1), cnt)
    assert np.all(np.abs(off[fin]) <= 32767)
    dc = np.where(fin, np.linalg.norm(off * step, axis=2), np.inf)
    inside = dk[:, K - 1] < rcap * (1 - 1e-3)
    assert np.all(cnt[inside] == K)
    tol = np.sqrt(3) * step / 2 + 1e-6 * rcap
    assert np.all(np.abs(np.sort(dc[inside], axis=1) - dk[inside, :K]) <= tol)
    # the decoded candidates are cloud points (up to the offset rounding)
    m = np.nonzero(inside)[0][:2000]
    for i in m[:200]:
        got = x0[i] + off[i, :cnt[i]] * step
        dd, _ = kt.query(got)
        assert np.all(dd <= tol)
    tight = dk[:, K] < rcap * (1 - 1e-3)
    assert np.all(kd[tight] >= dk[tight, K] - 2 * step - 1e-6 * rcap)
    return f


def test_field_records_uploaded_and_built_trees():
    z = load_golden("cfg0.npz")
    t = golden_tree(z, "")
    tree = upload(t)
    check_field(tree, W.cfg0_cloud())
    cloud = W.cfg1_cloud()
    tree1 = P.construct(P.PointCloud(cloud), P.BuildParams(0.02, 0.08))
    f = check_field(tree1, cloud)
    assert f["h"] < 0.02  # about 2 M cells over the tabletop box
    # replicated trees rebuild the same field from the slab
    pytest.importorskip("torch")
    t2 = P.Capt.from_slab(tree1.slab_tensor())
    f2 = t2.clearance_field(cells=True, candidates=True)
    f1 = tree1.clearance_field(cells=True, candidates=True)
    assert np.array_equal(f2["cells"], f1["cells"])
    assert np.array_equal(f2["candidates"], f1["candidates"])


def check_block_table(tree, cloud, n=400000, seed=0):
    """Every block entry q certifies q * step <= the float64 distance from the
    cloud to any centre whose computed cell lies in the block; sampled
    centres (uniform over the grid, and clustered near block faces) are
    checked against every block their computed cell could fall in."""
    from scipy.spatial import cKDTree
    f = tree.clearance_field()
    b = tree.field_blocks()
    assert b is not None
    tab, sh, step = b["table"], b["shift"], float(b["step"])
    nz, ny, nx = f["shape"]
    assert tab.shape == (-(-nz >> sh), -(-ny >> sh), -(-nx >> sh))
    assert step > 0 and (np.frexp(step)[0] == 0.5)  # a power of two
    h = float(f["h"])
    c0 = f["c0"].astype(np.float64)
    rng = np.random.default_rng(seed)
    dims = np.array([nx, ny, nz])
    t = rng.uniform(-0.5, dims - 0.5, (n, 3))
    # half of them on block faces (+-1e-4 cells)
    B = 1 << sh
    face = rng.integers(0, 3, n // 2)
    edge = (rng.integers(0, dims.max() // B + 1, n // 2) * B - 0.5)
    t[np.arange(n // 2), face] = np.clip(edge + rng.uniform(-1e-4, 1e-4, n // 2), -0.5,
                                         dims[face] - 0.5)
    c = (c0 + t * h).astype(np.float32).astype(np.float64)
    d, _ = cKDTree(np.unique(cloud.astype(np.float32), axis=0).astype(np.float64)).query(c)
    tt = (c - c0) / h
    worst = np.inf
    for dx in (-1e-3, 0.0, 1e-3):
        cell = np.clip(np.rint(tt + dx), 0, dims - 1).astype(np.int64)
        blk = cell >> sh
        q = tab[blk[:, 2], blk[:, 1], blk[:, 0]].astype(np.float64)
        assert np.all(q * step <= d), "block bound above a nearest-point distance"
        worst = min(worst, float(np.min(d - q * step)))
    return float((tab > 0).mean())


def test_field_block_table_bounds():
    for cloud, band in ((W.cfg1_cloud(), (0.02, 0.08)), (W.cfg3_cloud(n=65536, seed=11), (0.01, 0.1)),
                        (W.cfg0_cloud(), (0.01, 0.08))):
        tree = P.construct(P.PointCloud(cloud), P.BuildParams(*band))
        assert check_block_table(tree, cloud) > 0.05


def test_field_golden_masks_and_groups():
    z = load_golden("queries.npz")
    for name in z["names"]:
        pts = z[f"{name}/points"]
        rmin, rmax = z[f"{name}/band"]
        t = O.construct(pts, rmin, rmax)
        if t["k"] != 3:
            continue
        tree = upload(t)
        c, r = z[f"{name}/centers"], z[f"{name}/radii"]
        n = len(r)
        exp = np.unpackbits(z[f"{name}/mask"])[:n].astype(bool)
        assert np.array_equal(q(tree, c, r), exp), name
        nopre = np.unpackbits(z[f"{name}/mask_nopre"])[:n].astype(bool)
        assert np.array_equal(q(tree, c, r, prefilter=False), nopre), name
        lane = np.unpackbits(z[f"{name}/lane_mask"])[:n].astype(bool)
        gb = np.unpackbits(z[f"{name}/group8"])[: n // 8].astype(bool)
        assert np.array_equal(q(tree, c, r, 8, lane.astype(np.uint8)), gb), name


def test_field_cfg0_golden_and_full_batch():
    z = load_golden("cfg0.npz")
    t = golden_tree(z, "")
    tree = upload(t)
    n = int(z["n_queries"][0])
    c, r = W.cfg0_queries()
    assert np.array_equal(q(tree, c[:n], r[:n]), np.unpackbits(z["mask"])[:n].astype(bool))
    assert np.array_equal(q(tree, c, r), O.collides_many(t, c, r))
    # the default (auto) path is the field pipeline for fp32 input
    assert np.array_equal(P.collides_many(tree, c, r), O.collides_many(t, c, r))


@pytest.mark.parametrize("L", [1, 2, 4, 8, 16, 32])
def test_field_tabletop_groups_and_lane_masks(L):
    cloud = W.cfg1_cloud()
    tree = P.construct(P.PointCloud(cloud), P.BuildParams(0.02, 0.08))
    t = O.tree_from(tree)
    c, r = W.cfg1_queries(cloud, n_groups=1 << 16, seed=11)
    rng = np.random.default_rng(L)
    mask = (rng.uniform(size=len(r)) > 0.2).astype(np.uint8)
    exp = O.collides_groups(t, c, r, L, mask.astype(bool))
    assert np.array_equal(q(tree, c, r, L, mask), exp)
    # unmasked: the specialised K0 paths (L = 1, 8) and the generic one
    assert np.array_equal(q(tree, c, r, L), O.collides_groups(t, c, r, L))
    if L == 1:
        assert np.array_equal(q(tree, c, r), O.brute_collides_many(cloud, c, r))


@pytest.mark.parametrize("L", [4, 8, 16])
def test_field_group_kernel_tails_and_edge_radii(L):
    # the strided K0 with lane groups (k_resolve1<L>): a ragged last chunk
    # (its group bits are a 4-, 2- or 1-byte store), chunks with out-of-band
    # and NaN radii (the body with the band bookkeeping; check_radii off: the
    # reference's own semantics for those lanes), first_bad with check_radii
    cloud = W.cfg1_cloud()
    tree = P.construct(P.PointCloud(cloud), P.BuildParams(0.02, 0.08))
    t = O.tree_from(tree)
    for n_groups in (65536 + 37, 16385, 8192 + 1):
        c, r = W.cfg1_queries(cloud, n_groups=n_groups, lane_width=L, seed=5 + L)
        assert np.array_equal(q(tree, c, r, L), O.collides_groups(t, c, r, L))
        r2 = r.copy()
        r2[3::1013] = np.float32(0.5)  # out of band
        r2[7::2029] = np.nan
        r2[11::4051] = np.float32(0.001)
        assert np.array_equal(q(tree, c, r2, L), O.collides_groups(t, c, r2, L))
        bits, bad = q(tree, c, r2, L, check=True)
        flagged = ((r2.astype(np.float64) < 0.02) | (r2.astype(np.float64) > 0.08)) & ~np.isnan(r2)
        assert bad == int(np.argmax(flagged))


def test_field_tangent_spheres():
    # radius = the float32 image of the exact nearest-point distance, and one
    # ulp either side: every sphere sits on the certificates' decision edge
    from scipy.spatial import cKDTree
    rng = np.random.default_rng(23)
    pts = rng.uniform(0, 1, (4096, 3)).astype(np.float32)
    t = O.construct(pts, 0.01, 0.08)
    tree = upload(t)
    n = 1 << 17
    idx = rng.integers(0, len(pts), n)
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    r0 = rng.uniform(0.011, 0.079, n)
    c = (pts[idx].astype(np.float64) + d * r0[:, None]).astype(np.float32)
    nn, _ = cKDTree(pts.astype(np.float64)).query(c.astype(np.float64))
    r = np.float32(nn)
    for rr in (r, np.nextafter(r, np.float32(0)), np.nextafter(r, np.float32(1))):
        rr = W.clamp_radii(rr.astype(np.float32), 0.01, 0.08)
        exp = O.collides_many(t, c, rr)
        got = q(tree, c, rr)
        assert np.array_equal(got, exp)
        assert np.array_equal(got, O.brute_collides_many(pts, c, rr))


def test_field_edge_inputs():
    # out-of-band radii with check_radii=False (the reference's own semantics,
    # not the brute-force ones), NaN radii, non-finite centres, centres far
    # outside the cloud's box, a batch that is not a multiple of 32
    rng = np.random.default_rng(31)
    pts = rng.uniform(-1, 1, (5000, 3)).astype(np.float32)
    t = O.construct(pts, 0.02, 0.08)
    tree = upload(t)
    n = 200003
    c = rng.uniform(-1.3, 1.3, (n, 3)).astype(np.float32)
    r = rng.uniform(0.0, 0.2, n).astype(np.float32)  # many outside [0.02, 0.08]
    c[::997, 0] = np.nan
    c[5::991, 2] = np.inf
    c[7::983] = np.float32(1e30)
    r[11::977] = np.nan
    r[13::971] = np.inf
    r[17::89] *= -1  # negative radii collide like their magnitude (d^2 <= r*r)
    exp = O.collides_many(t, c, r)
    assert np.array_equal(q(tree, c, r), exp)
    assert np.array_equal(q(tree, c, r, prefilter=False), O.collides_many(t, c, r, False))
    # check_radii: the first out-of-band index is reported (NaN is not flagged)
    bits, bad = q(tree, c, r, check=True)
    inb = (r.astype(np.float64) >= 0.02) & (r.astype(np.float64) <= 0.08)
    flagged = ~inb & ~np.isnan(r)
    assert bad == int(np.argmax(flagged))


def test_field_dense_gaussians():
    cloud = W.cfg3_cloud(n=32768, n_comp=8, seed=5)
    t = O.construct(cloud, 0.01, 0.1)
    tree = upload(t)
    check_field(tree, cloud, sample=50000)
    c, r = W.cfg3_queries(1 << 19, seed=7)
    assert np.array_equal(q(tree, c, r), O.collides_many(t, c, r))


def test_field_degenerate_clouds():
    # one point; a flat plane (zero z extent); duplicates; a line
    rng = np.random.default_rng(3)
    clouds = [np.array([[0.25, -0.5, 1.0]], np.float32),
              np.c_[rng.uniform(-1, 1, (3000, 2)), np.zeros(3000)].astype(np.float32),
              np.repeat(rng.uniform(0, 1, (500, 3)), 3, axis=0).astype(np.float32),
              # 40 copies of every point: the candidate lists fill with copies
              # of one point, so their bound certifies little and many
              # spheres take the tree path
              np.repeat(rng.uniform(0, 1, (100, 3)), 40, axis=0).astype(np.float32),
              np.c_[np.linspace(0, 1, 2000), np.zeros(2000), np.zeros(2000)].astype(np.float32)]
    for i, cloud in enumerate(clouds):
        t = O.construct(cloud, 0.01, 0.05)
        tree = upload(t)
        check_field(tree, cloud, sample=20000)
        lo, hi = cloud.min(0) - 0.1, cloud.max(0) + 0.1
        c = rng.uniform(lo, hi, (100000, 3)).astype(np.float32)
        r = W.clamp_radii(rng.uniform(0.01, 0.05, 100000).astype(np.float32), 0.01, 0.05)
        assert np.array_equal(q(tree, c, r), O.collides_many(t, c, r)), i
        assert np.array_equal(q(tree, c, r, 8), O.collides_groups(t, c, r, 8)), i


@pytest.mark.parametrize("L", [1, 8])
def test_field_f64_inputs_split_on_device(L):
    # float64 batches: the spheres whose values are fp32 values take the
    # field pipeline, the others (perturbed centres or radii, huge values)
    # the float64 path, on the device; masks and the first out-of-band
    # index (an inexact radius) come out as the reference's
    cloud = W.cfg1_cloud()
    t = O.construct(cloud, 0.02, 0.08)
    tree = upload(t)
    c, r = W.cfg1_queries(cloud, n_groups=1 << 15, seed=41)
    c64, r64 = c.astype(np.float64), r.astype(np.float64)
    rng = np.random.default_rng(42)
    n = len(r)
    pick = rng.choice(n, n // 10, replace=False)
    c64[pick[: len(pick) // 2], 1] += 1e-9
    r64[pick[len(pick) // 2:]] *= 1 + 1e-12
    c64[pick[:50], 0] = 1e300
    mask = (rng.uniform(size=n) > 0.1).astype(np.uint8)
    for m in (None, mask):
        exp = (O.collides_many(t, c64, r64) if L == 1 and m is None else
               O.collides_groups(t, c64, r64, L, None if m is None else m.astype(bool)))
        assert np.array_equal(q(tree, c64, r64, L, m), exp)
        assert np.array_equal(q(tree, c64, r64, L, m, mode=0), exp)
    # check_radii: an inexact out-of-band radius is the first bad index
    r_bad = r64.copy()
    r_bad[777] = 0.08 + 1e-12
    r_bad[5000] = 0.5
    bits, bad = q(tree, c64, r_bad, L, check=True, mode=0)
    assert bad == 777


def test_stage_timing_abi():
    # capt_stage_timing / capt_stage_times: events around K0 and the list
    # stage of field-pipeline calls (bench.py's roofline split)
    import ctypes
    torch = pytest.importorskip("torch")
    z = load_golden("cfg0.npz")
    tree = upload(golden_tree(z, ""))
    c, r = W.cfg0_queries(1 << 18)
    cd, rd = torch.from_numpy(c).cuda(), torch.from_numpy(r).cuda()
    L = _lib.lib()
    ms = (ctypes.c_double * 3)()
    calls = ctypes.c_int64(0)
    assert L.capt_stage_timing(1) == 0
    for _ in range(3):  # (forced: below 1 M spheres auto mode takes the fused small kernel)
        P.query_bits(tree, cd, rd, 1, mode=FIELD)
    torch.cuda.synchronize()
    assert L.capt_stage_times(ms, ctypes.byref(calls)) == 0
    assert calls.value == 3
    assert ms[0] > 0 and ms[1] > 0 and abs(ms[2] - ms[0] - ms[1]) < 1e-6
    # the record is cleared by the read; disabled timing records nothing
    assert L.capt_stage_times(ms, ctypes.byref(calls)) == 0 and calls.value == 0
    assert L.capt_stage_timing(0) == 0
    P.query_bits(tree, cd, rd, 1, mode=FIELD)
    torch.cuda.synchronize()
    assert L.capt_stage_times(ms, ctypes.byref(calls)) == 0 and calls.value == 0
    exp = O.collides_many(golden_tree(z, ""), c, r)
    got = P.collides_many(tree, c, r)
    assert np.array_equal(got, exp)


def test_field_unaligned_inputs_and_f64_exact():
    # views 12 / 4 bytes into their buffers (no 128-bit loads: the scalar K0
    # path), and float64 arrays holding fp32 values (converted, fp32 path)
    z = load_golden("cfg0.npz")
    t = golden_tree(z, "")
    tree = upload(t)
    c, r = W.cfg0_queries((1 << 17) + 1)
    cu, ru = c[1:], r[1:]
    assert cu.ctypes.data % 16 and ru.ctypes.data % 16
    exp = O.collides_many(t, cu, ru)
    assert np.array_equal(q(tree, cu, ru), exp)
    assert np.array_equal(P.collides_many(tree, cu.astype(np.float64), ru.astype(np.float64)), exp)


def test_field_room_scale_cells_wider_than_r_min():
    # an 8 x 8 x 3 m room: the ~2 M-cell field has cells of 4.8 cm, wider
    # than r_min = 1 cm, so the certificates decide less and more spheres
    # take the list stage (candidate records, bucket scan); verdicts stay
    # the reference's
    cloud = W.room_cloud(n=100000, seed=9)
    tree = P.construct(P.PointCloud(cloud), P.BuildParams(0.01, 0.08))
    f = tree.clearance_field()
    assert f["h"] > 0.01
    t = O.construct(cloud, 0.01, 0.08)
    c, r = W.room_queries(cloud, n=1 << 20, seed=10)
    assert np.array_equal(q(tree, c, r, mode=0), O.collides_many(t, c, r))
    assert np.array_equal(q(tree, c, r, 8, mode=0), O.collides_groups(t, c, r, 8))


@pytest.mark.parametrize("L", [1, 2, 8, 32])
def test_small_batch_fused_kernel(L):
    # batches below CAPT_SMALL_BATCH take one fused kernel (k_resolve_small):
    # K0's certificates, then per open sphere the candidate record, the
    # bucket scan or the tree path, whole verdict words; sizes with partial
    # last words, lane masks, out-of-band and non-finite spheres (check_radii
    # off: the reference's semantics), the first bad radius (check_radii on)
    cloud = W.cfg1_cloud()
    t = O.construct(cloud, 0.02, 0.08)
    tree = upload(t)
    rng = np.random.default_rng(100 + L)
    for groups in (1, 3, 37, 1000, 8191):
        c, r = W.cfg1_queries(cloud, n_groups=groups, lane_width=L, seed=groups)
        c = c.copy()
        r = r.copy()
        k = len(r)
        if k > 16:
            c[3, 0] = np.nan
            c[5, 1] = np.inf
            r[7] = 0.5        # out of band
            r[11] = np.nan
        exp = O.collides_groups(t, c, r, L)
        assert np.array_equal(q(tree, c, r, L, mode=0), exp), groups
        m = (rng.uniform(size=k) > 0.3).astype(np.uint8)
        assert np.array_equal(q(tree, c, r, L, m, mode=0),
                              O.collides_groups(t, c, r, L, m.astype(bool))), groups
        if k > 16:
            bits, bad = q(tree, c, r, L, check=True, mode=0)
            assert bad == 7
