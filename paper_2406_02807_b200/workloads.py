"""Seeded synthetic inputs for the five BASELINE.json configurations.

These stand in for the paper's MotionBenchMaker clouds, planner traces and
RealSense captures, none of which are available
here.  Everything is generated with ``numpy.random.default_rng(seed)`` in
float64 and cast to float32; the same fp32 arrays feed the GPU path and the
CPU oracle.  Choices the configuration text leaves open are fixed here and
recorded in DESIGN.md (section "Workloads").

Radii are clamped into the double exactness band after the fp32 cast
(SURVEY 8d): fp32(0.01), fp32(0.02), fp32(0.08) lie below the double band
edges and fp32(0.1) above, and the reference checks the band in double
(query.py:30-34).  The reference's own generator keeps a margin for the same
reason (synth.py:98-101).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["CONFIGS", "f32_band", "clamp_radii", "cfg0_cloud", "cfg0_queries",
           "tabletop_scene", "cfg1_cloud", "cfg1_queries", "cfg2_raw_cloud",
           "cfg2_queries", "cfg3_cloud", "cfg3_queries", "cfg4_queries",
           "uniform_queries", "room_cloud", "room_queries"]


@dataclass(frozen=True)
class ConfigSpec:
    name: str
    r_min: float
    r_max: float
    n_queries: int       # spheres (groups x 8 for config 1)
    lane_width: int      # 1 = per-sphere verdicts, 8 = any-collision groups


CONFIGS = {
    0: ConfigSpec("cfg0-uniform-2048", 0.01, 0.08, 1 << 20, 1),
    1: ConfigSpec("cfg1-tabletop-16384-groups8", 0.02, 0.08, (4 << 20) * 8, 8),
    2: ConfigSpec("cfg2-depthcam-filtered", 0.01, 0.08, 16 << 20, 1),
    3: ConfigSpec("cfg3-gaussians-262144", 0.01, 0.1, 64 << 20, 1),
    4: ConfigSpec("cfg4-sweep-tabletop", 0.02, 0.08, 0, 1),
}


def f32_band(r_min: float, r_max: float) -> tuple[np.float32, np.float32]:
    """Smallest fp32 >= r_min and largest fp32 <= r_max (double compares)."""
    lo = np.float32(r_min)
    if float(lo) < r_min:
        lo = np.nextafter(lo, np.float32(np.inf))
    hi = np.float32(r_max)
    if float(hi) > r_max:
        hi = np.nextafter(hi, np.float32(0))
    return np.float32(lo), np.float32(hi)


def clamp_radii(r: np.ndarray, r_min: float, r_max: float) -> np.ndarray:
    lo, hi = f32_band(r_min, r_max)
    return np.clip(np.asarray(r, np.float32), lo, hi).astype(np.float32)


def uniform_queries(rng, n: int, lo, hi, r_min: float, r_max: float):
    """(centers (n,3) fp32, radii (n,) fp32): centers U[lo,hi], radii U[r_min,r_max]."""
    c = rng.uniform(lo, hi, size=(n, 3)).astype(np.float32)
    r = clamp_radii(rng.uniform(r_min, r_max, size=n).astype(np.float32), r_min, r_max)
    return c, r


# --------------------------------------------------------------------------
# config 0: uniform cube (runs on the CPU reference)
# --------------------------------------------------------------------------

def cfg0_cloud(n: int = 2048, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.uniform(-1.0, 1.0, size=(n, 3)).astype(np.float32)


def cfg0_queries(n: int = 1 << 20, seed: int = 1):
    rng = np.random.default_rng(seed)
    return uniform_queries(rng, n, -1.1, 1.1, 0.01, 0.08)


# --------------------------------------------------------------------------
# config 1: tabletop box scene
# --------------------------------------------------------------------------

TABLE_HALF = 0.75  # 1.5 x 1.5 m table, centred on the origin, top at z = 0


def tabletop_scene(seed: int = 1, n_boxes: int = 20):
    """Axis-aligned boxes (lo, hi) resting on the table.  Sides U[0.05, 0.4];
    footprints fully on the table."""
    rng = np.random.default_rng(seed)
    sides = rng.uniform(0.05, 0.4, size=(n_boxes, 3))
    cx = rng.uniform(-TABLE_HALF + sides[:, 0] / 2, TABLE_HALF - sides[:, 0] / 2)
    cy = rng.uniform(-TABLE_HALF + sides[:, 1] / 2, TABLE_HALF - sides[:, 1] / 2)
    lo = np.stack([cx - sides[:, 0] / 2, cy - sides[:, 1] / 2, np.zeros(n_boxes)], 1)
    hi = lo + sides
    return lo, hi, rng


def _scene_rects(box_lo, box_hi):
    """Table rectangle + the 5 exposed faces of every box (bottom faces rest on
    the table and are not sampled).  Each rect is (origin, u, v) like the
    reference's rectangle sampler (synth.py:36-47)."""
    t = TABLE_HALF
    rects = [(np.array([-t, -t, 0.0]), np.array([2 * t, 0, 0.0]), np.array([0, 2 * t, 0.0]))]
    for lo, hi in zip(box_lo, box_hi):
        d = hi - lo
        ex, ey, ez = np.diag(d)
        rects += [(lo + ez, ex, ey),            # top
                  (lo, ex, ez), (lo + ey, ex, ez),  # y faces
                  (lo, ey, ez), (lo + ex, ey, ez)]  # x faces
    return rects


def cfg1_cloud(n: int = 16384, seed: int = 1, noise: float = 0.002) -> np.ndarray:
    box_lo, box_hi, rng = tabletop_scene(seed)
    rects = _scene_rects(box_lo, box_hi)
    areas = np.array([np.linalg.norm(np.cross(u, v)) for _, u, v in rects])
    counts = rng.multinomial(n, areas / areas.sum())
    chunks = []
    for (o, u, v), m in zip(rects, counts):
        if m == 0:
            continue
        a = rng.uniform(size=(m, 1))
        b = rng.uniform(size=(m, 1))
        chunks.append(o + a * u + b * v)
    pts = np.concatenate(chunks, 0)
    pts = pts + rng.normal(0.0, noise, size=pts.shape)
    return pts.astype(np.float32)


def cfg1_queries(cloud: np.ndarray, n_groups: int = 4 << 20, lane_width: int = 8,
                 seed: int = 101, offset: float = 0.05):
    """Spatially-correlated groups: base centre U(scene AABB), per-axis offsets
    U[-offset, offset], radii U[0.02, 0.08].  Returns (centers (G*L,3),
    radii (G*L,)) with group g occupying rows [g*L, (g+1)*L)."""
    rng = np.random.default_rng(seed)
    lo = cloud.min(0).astype(np.float64)
    hi = cloud.max(0).astype(np.float64)
    base = rng.uniform(lo, hi, size=(n_groups, 1, 3))
    off = rng.uniform(-offset, offset, size=(n_groups, lane_width, 3))
    c = (base + off).reshape(-1, 3).astype(np.float32)
    r = clamp_radii(rng.uniform(0.02, 0.08, size=n_groups * lane_width).astype(np.float32),
                    0.02, 0.08)
    return c, r


# --------------------------------------------------------------------------
# config 2: synthetic depth camera over the config-1 scene
# --------------------------------------------------------------------------

CAMERA = dict(width=640, height=480, fx=525.0, fy=525.0, cx=320.0, cy=240.0,
              eye=(0.0, -TABLE_HALF, 1.2), target=(0.0, 0.0, 0.0),
              near=0.3, far=3.0, depth_noise=0.005)


def _camera_basis(eye, target):
    eye = np.asarray(eye, float)
    fwd = np.asarray(target, float) - eye
    fwd /= np.linalg.norm(fwd)
    up = np.array([0.0, 0.0, 1.0])
    right = np.cross(fwd, up)
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    return eye, right, down, fwd


def _ray_aabb(o, d, lo, hi):
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / d
        t1 = (lo - o) * inv
        t2 = (hi - o) * inv
    tmin = np.nanmax(np.minimum(t1, t2), axis=1)
    tmax = np.nanmin(np.maximum(t1, t2), axis=1)
    hit = (tmax >= np.maximum(tmin, 0.0))
    return np.where(hit, tmin, np.inf)


def cfg2_raw_cloud(seed: int = 2) -> np.ndarray:
    """Ray-cast the config-1 scene (table + boxes, box layout seed 1) from the
    CAMERA pinhole; depth = camera-z distance, valid in [near, far], scaled by
    N(1, depth_noise)."""
    cam = CAMERA
    box_lo, box_hi, _ = tabletop_scene(1)
    eye, right, down, fwd = _camera_basis(cam["eye"], cam["target"])
    v, u = np.mgrid[0:cam["height"], 0:cam["width"]]
    x = (u.ravel() + 0.0 - cam["cx"]) / cam["fx"]
    y = (v.ravel() + 0.0 - cam["cy"]) / cam["fy"]
    d = x[:, None] * right + y[:, None] * down + fwd  # camera-z component == 1
    o = np.broadcast_to(eye, d.shape)
    # table top plane z = 0 restricted to the table square
    with np.errstate(divide="ignore", invalid="ignore"):
        t_plane = -eye[2] / d[:, 2]
    hp = o + t_plane[:, None] * d
    ok = (t_plane > 0) & (np.abs(hp[:, 0]) <= TABLE_HALF) & (np.abs(hp[:, 1]) <= TABLE_HALF)
    t = np.where(ok, t_plane, np.inf)
    for lo, hi in zip(box_lo, box_hi):
        t = np.minimum(t, _ray_aabb(o, d, lo, hi))
    depth = t  # |d_z| == 1 in the camera frame
    valid = np.isfinite(depth) & (depth >= cam["near"]) & (depth <= cam["far"])
    rng = np.random.default_rng(seed)
    noise = rng.normal(1.0, cam["depth_noise"], size=depth.shape)
    depth = depth * noise
    pts = eye + d[valid] * depth[valid, None]
    return pts.astype(np.float32)


def cfg2_queries(filtered: np.ndarray, n: int = 16 << 20, seed: int = 102):
    rng = np.random.default_rng(seed)
    lo = filtered.min(0).astype(np.float64)
    hi = filtered.max(0).astype(np.float64)
    pad = 0.1 * (hi - lo)
    return uniform_queries(rng, n, lo - pad, hi + pad, 0.01, 0.08)


# --------------------------------------------------------------------------
# config 3: large dense Gaussian-mixture cloud
# --------------------------------------------------------------------------

def cfg3_cloud(n: int = 262144, n_comp: int = 64, seed: int = 3) -> np.ndarray:
    """Equal-weight mixture (n / n_comp points per component)."""
    rng = np.random.default_rng(seed)
    mu = rng.uniform(-1.0, 1.0, size=(n_comp, 3))
    sig = rng.uniform(0.01, 0.1, size=(n_comp, 3))
    comp = np.repeat(np.arange(n_comp), n // n_comp)
    pts = mu[comp] + rng.normal(size=(len(comp), 3)) * sig[comp]
    return pts.astype(np.float32)


def cfg3_queries(n: int = 64 << 20, seed: int = 103):
    rng = np.random.default_rng(seed)
    return uniform_queries(rng, n, -1.2, 1.2, 0.01, 0.1)


# --------------------------------------------------------------------------
# config 4: collision-rate x batch-size sweep on the config-1 cloud
# --------------------------------------------------------------------------

def cfg4_queries(cloud: np.ndarray, n: int, rate: float, seed: int = 104,
                 r_min: float = 0.02, r_max: float = 0.08):
    """Per-sphere Bernoulli(rate) label; colliding centres = random cloud point
    + random direction * U[0, 0.9) * r (synth.py:104-111); free centres are
    rejection-sampled with fp64 nearest-neighbour distance > r * (1 + 1e-6)
    after the fp32 cast (synth.py:114-131).  Radii U[0.02, 0.08]: the cloud's
    tree band is [0.02, 0.08] (config text says U[0.01, 0.08], which the
    reference would reject; DESIGN.md records the choice)."""
    from scipy.spatial import cKDTree

    rng = np.random.default_rng(seed)
    pts = cloud.astype(np.float64)
    r = clamp_radii(rng.uniform(r_min, r_max, size=n).astype(np.float32), r_min, r_max)
    label = rng.uniform(size=n) < rate
    c = np.empty((n, 3), np.float32)
    hit_idx = np.nonzero(label)[0]
    if len(hit_idx):
        j = rng.integers(0, len(pts), size=len(hit_idx))
        dirs = rng.normal(size=(len(hit_idx), 3))
        dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
        off = dirs * (rng.uniform(0.0, 0.9, size=len(hit_idx)) * r[hit_idx])[:, None]
        c[hit_idx] = (pts[j] + off).astype(np.float32)
    free_idx = np.nonzero(~label)[0]
    if len(free_idx):
        kd = cKDTree(pts)
        lo = pts.min(0) - 3 * r_max
        hi = pts.max(0) + 3 * r_max
        todo = free_idx
        while len(todo):
            cand = rng.uniform(lo, hi, size=(len(todo), 3)).astype(np.float32)
            dist, _ = kd.query(cand.astype(np.float64))
            good = dist > r[todo].astype(np.float64) * (1.0 + 1e-6)
            c[todo[good]] = cand[good]
            todo = todo[~good]
    return c, r, label


# --------------------------------------------------------------------------
# room-scale stress case (not a BASELINE config): the clearance field's cell
# edge grows with the scene, so this covers the regime where a fixed cell
# budget would leave cells wider than r_min
# --------------------------------------------------------------------------

def room_cloud(n: int = 200000, seed: int = 7, size=(8.0, 8.0, 3.0), n_boxes: int = 40,
               noise: float = 0.002) -> np.ndarray:
    """Points on the floor, walls and ceiling of a size[0] x size[1] x size[2]
    room plus n_boxes furniture boxes on the floor, area-weighted, N(0, noise)."""
    rng = np.random.default_rng(seed)
    X, Y, Z = size
    rects = [(np.array([0.0, 0, 0]), np.array([X, 0, 0.0]), np.array([0, Y, 0.0])),
             (np.array([0.0, 0, Z]), np.array([X, 0, 0.0]), np.array([0, Y, 0.0])),
             (np.array([0.0, 0, 0]), np.array([X, 0, 0.0]), np.array([0, 0, Z])),
             (np.array([0.0, Y, 0]), np.array([X, 0, 0.0]), np.array([0, 0, Z])),
             (np.array([0.0, 0, 0]), np.array([0, Y, 0.0]), np.array([0, 0, Z])),
             (np.array([X, 0, 0.0]), np.array([0, Y, 0.0]), np.array([0, 0, Z]))]
    sides = rng.uniform(0.3, 1.5, size=(n_boxes, 3))
    lo = np.stack([rng.uniform(0, X - sides[:, 0]), rng.uniform(0, Y - sides[:, 1]),
                   np.zeros(n_boxes)], 1)
    for l, d in zip(lo, sides):
        ex, ey, ez = np.diag(d)
        rects += [(l + ez, ex, ey), (l, ex, ez), (l + ey, ex, ez), (l, ey, ez), (l + ex, ey, ez)]
    areas = np.array([np.linalg.norm(np.cross(u, v)) for _, u, v in rects])
    counts = rng.multinomial(n, areas / areas.sum())
    chunks = [o + rng.uniform(size=(m, 1)) * u + rng.uniform(size=(m, 1)) * v
              for (o, u, v), m in zip(rects, counts) if m]
    pts = np.concatenate(chunks, 0) + rng.normal(0.0, noise, size=(n, 3))
    return pts.astype(np.float32)


def room_queries(cloud: np.ndarray, n: int = 16 << 20, seed: int = 8, r_min: float = 0.01,
                 r_max: float = 0.08):
    rng = np.random.default_rng(seed)
    return uniform_queries(rng, n, cloud.min(0).astype(np.float64),
                           cloud.max(0).astype(np.float64), r_min, r_max)
