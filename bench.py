"""Benchmark: CAPT batched sphere-collision queries on B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C]
                    [--scaling auto|weak|strong] [--impl ours|reference] [--sweep]

Default workload = BASELINE.json configs[3], the config BASELINE's metric is
quoted "at 1/2/4/8 B200" on and the largest single-GPU configuration: a
262,144-point Gaussian-mixture cloud (CAPT r_min 0.01 / r_max 0.1, a 5.7 GB
tree) queried with 67,108,864 independent spheres, the batch split across
the GPUs (strong scaling, the tree replicated by one NCCL broadcast of its
device slab, the counters summed by one NCCL all-reduce; no data-path
collective).  ``--config 1`` is the tabletop scene with 4M groups of 8
spheres (edge-validation early exit, query.py:126-167), ``--config 2`` the
depth-camera pipeline (device filter and build timed separately, then the
16M-sphere query), ``--config 0`` the uniform cube, ``--sweep`` the config-4
batch-size x collision-rate grid.

One "step" = one capt_query over the rank's shard with inputs resident in
HBM (16 B/sphere: 1 GB per config-3 step, > the 126 MB L2, so no flush is
needed).  After the timed region the whole job's verdict words are gathered
on rank 0 and compared with the CPU oracle (oracle/, a C restatement of
captree's construct / collides_many / collides_batch), the device tree with
the oracle's construct of the same cloud; the line carries the mismatch
counts and the boundary-sphere count (|d^2 - r^2| < 1e-6).
``e2e`` times the same batch through the C-ABI with host buffers, the
host->device copies and the verdict device->host copy inside the region.

``--impl reference`` times the reference algorithm on the host CPU (the
oracle port, every host thread) on the same config; rank 0 alone runs it.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2406_02807_b200 import workloads as W  # noqa: E402

METRIC = "CAPT sphere collision queries/sec at 1/2/4/8 B200; % of roofline; vs CPU ref"
UNIT = "queries/s"
FLOP_PER_TEST = 8  # 3 sub + 3 mul + 2 add
CAND_RECORD_BYTES = 192  # kCandWords x 4 (capt_internal.cuh)
# the paper's single-core C++ figures for one 307,200-point frame
# (ref PAPER.md:766-770): filter 6.944 ms, CAPT build 30.373 ms
PAPER_FILTER_MS, PAPER_BUILD_MS = 6.944, 30.373


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=3, choices=[0, 1, 2, 3])
    ap.add_argument("--scaling", default="auto", choices=["auto", "weak", "strong"],
                    help="auto: strong for config 3 (BASELINE: 'query batch split across "
                         "1/2/4/8 GPUs'), weak otherwise")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="auto", choices=["auto", "direct", "binned"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--sweep", action="store_true",
                    help="config-4 batch-size x collision-rate sweep (one JSON object)")
    ap.add_argument("--sweep-max-exp", type=int, default=14,
                    help="largest batch is 4^this spheres (14 -> 268M, ~4.3 GB)")
    a = ap.parse_args()
    if a.scaling == "auto":
        a.scaling = "strong" if a.config == 3 else "weak"
    return a


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# --------------------------------------------------------------------------
# workloads
# --------------------------------------------------------------------------

DESC = {
    0: "cfg0: 2,048 uniform points (r 0.01/0.08), 1,048,576 independent spheres",
    1: "cfg1: tabletop scene (16,384 pts, r 0.02/0.08), 4,194,304 groups x 8 spheres, "
       "one any-collision bit per group",
    2: "cfg2: depth-camera frame of the tabletop (640x480 pinhole, 254,438 pts) -> Z-order "
       "filter r_f 0.01 -> CAPT r 0.01/0.08, 16,777,216 spheres",
    3: "cfg3: 262,144-pt mixture of 64 anisotropic Gaussians (r 0.01/0.1, 5.7 GB tree), "
       "67,108,864 spheres",
}


def cloud_for(cfg: int, filtered=None):
    if cfg == 0:
        return W.cfg0_cloud()
    if cfg == 1:
        return W.cfg1_cloud()
    if cfg == 2:
        return filtered
    return W.cfg3_cloud()


def batch_for(cfg: int, seed_rank: int, cloud):
    """(centers, radii) of one batch (config spec size); weak scaling gives
    rank r the seed offset 1000 r, strong scaling one global batch."""
    spec = W.CONFIGS[cfg]
    s = 1000 * seed_rank
    if cfg == 0:
        return W.cfg0_queries(spec.n_queries, seed=1 + s)
    if cfg == 1:
        return W.cfg1_queries(cloud, n_groups=spec.n_queries // 8, seed=101 + s)
    if cfg == 2:
        return W.cfg2_queries(cloud, n=spec.n_queries, seed=102 + s)
    return W.cfg3_queries(spec.n_queries, seed=103 + s)


def config_block(args, world: int) -> dict:
    """The ``config`` object, identical in both arms (no device results)."""
    spec = W.CONFIGS[args.config]
    n_job = spec.n_queries * (world if args.scaling == "weak" else 1)
    return {"workload": DESC[args.config], "config_index": args.config,
            "spheres_per_job": n_job, "lane_width": spec.lane_width,
            "unit_of_value": "sphere queries/s (groups/s = value / lane_width)",
            "r_min": spec.r_min, "r_max": spec.r_max, "scaling": args.scaling,
            "parallelism": f"dp{world} (query shards, tree replicated)",
            "l2": "inputs (16 B/sphere) exceed the 126 MB L2 at every config; no flush"}


# --------------------------------------------------------------------------
# clocks (NVML sampled during the timed region)
# --------------------------------------------------------------------------

class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 - no NVML: report nulls
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# --------------------------------------------------------------------------
# evidence files
# --------------------------------------------------------------------------

def profiled_traffic(config, kernel_substr):
    """DRAM bytes (read + write) of one launch of the kernel whose name
    contains ``kernel_substr``, from the newest committed ``ncu --set full``
    summary of this config (profiles/rNN_cfg<k>_ncu_full.json)."""
    pdir = os.path.join(ROOT, "profiles")
    cands = sorted(f for f in os.listdir(pdir)
                   if f.endswith(f"_cfg{config}_ncu_full.json") and f.startswith("r"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for fname in reversed(cands):
        for k in json.load(open(os.path.join(pdir, fname))):
            if kernel_substr not in k["kernel"]:
                continue
            tot = sum(float(k[f]) * scale.get(k.get(f + "_unit", "byte"), 1)
                      for f in ("dram_read", "dram_write"))
            return tot, f"profiles/{fname}: dram read+write of {k['kernel'].split('(')[0]}"
    return None, f"no ncu --set full capture of {kernel_substr} committed for config {config}"


# --------------------------------------------------------------------------
# CPU baselines (oracle port; the real reference on a prefix)
# --------------------------------------------------------------------------

def _oracle_run(O, tree_ref, c, r, L, threads):
    if L > 1:
        O.collides_groups(tree_ref, c, r, L, threads=threads)
    else:
        O.collides_many(tree_ref, c, r, threads=threads)


def median_rate(fn, n, reps=3):
    """The reference's protocol (ref bench.py:31-40): 1 warm-up + median of
    ``reps`` timed runs; returns (units/s, median seconds)."""
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    med = statistics.median(ts)
    return n / med, med


def size_sample(fn_n, L, target_s, n_max):
    """Largest n (multiple of L, <= n_max) that takes about target_s."""
    n = min(n_max, max(L, 1 << 14))
    n -= n % L
    t0 = time.perf_counter()
    fn_n(n)
    dt = max(time.perf_counter() - t0, 1e-6)
    m = int(min(n_max, n * target_s / dt))
    return max(L, m - m % L)


def cpu_port_rate(tree_ref, c, r, L, threads, target_s):
    from oracle import oracle as O
    c64, r64 = c.astype(np.float64), r.astype(np.float64)
    n = size_sample(lambda m: _oracle_run(O, tree_ref, c64[:m], r64[:m], L, threads), L,
                    target_s, len(r))
    rate, med = median_rate(lambda: _oracle_run(O, tree_ref, c64[:n], r64[:n], L, threads), n)
    return rate, n, med


def python_reference_rate(tree, c, r, L, target_s):
    """captree.collides_many (ref query.py:184-219), unmodified, from
    baseline/_ref (an offline pip install of /root/reference), on a prefix of
    the batch, 1 process; the tree is captree.Capt over this tree's arrays
    (ref tree.py:74-97).  None if baseline/_ref is absent."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "captree")):
        return None
    need = 48 * int(tree.stats().total_stored) + 64 * len(r)  # exported + captree's copies
    try:
        avail = int(open("/proc/meminfo").read().split("MemAvailable:")[1].split()[0]) * 1024
    except (OSError, IndexError, ValueError):
        avail = 0
    if need > avail // 4:
        return {"unavailable": f"captree.Capt copies of this tree need ~{need / 1e9:.0f} GB "
                               f"(host MemAvailable {avail / 1e9:.0f} GB); skipped"}
    if ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)
    try:
        import captree
    except Exception as exc:  # noqa: BLE001
        return {"unavailable": f"import captree failed: {exc}"}
    t = captree.Capt(tree.k, tree.n_points, tree.r_min, tree.r_max, tree.tests, tree.aff_lo,
                     tree.aff_hi, tree.offsets, tree.aff_values)
    c64, r64 = c.astype(np.float64), r.astype(np.float64)

    def run(m):
        v = captree.collides_many(t, c64[:m], r64[:m])
        if L > 1:
            v.reshape(-1, L).any(1)

    n = size_sample(run, L, target_s, len(r))
    rate, med = median_rate(lambda: run(n), n)
    return {"value": rate, "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"first {n} spheres, captree.collides_many from baseline/_ref (the "
                      f"unmodified reference, Python/numpy), 1 warm-up + median of 3 "
                      f"({med:.2f} s)"}


# --------------------------------------------------------------------------
# preprocessing (config 2): device filter + build, CPU references beside
# --------------------------------------------------------------------------

def preprocess_cfg2(P, dev, reps=10, cpu=True):
    import torch
    from paper_2406_02807_b200 import _lib
    raw = W.cfg2_raw_cloud()
    raw_d = torch.from_numpy(raw).to(dev)
    out_d = torch.empty_like(raw_d)
    n_out = ctypes.c_int64(0)
    lib = _lib.lib()
    r_f = 0.01

    def filt():
        _lib.check(lib.capt_filter_cloud(dev.index, 3, raw_d.data_ptr(), len(raw), r_f, 0, None,
                                         0.0, 0, out_d.data_ptr(), ctypes.byref(n_out),
                                         None), "capt_filter_cloud")

    def timed(fn):
        fn()
        torch.cuda.synchronize(dev)
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize(dev)
            ts.append((time.perf_counter() - t0) * 1e3)
        return statistics.median(ts), min(ts)

    f_med, f_min = timed(filt)
    filtered_d = out_d[: n_out.value].contiguous()
    params = P.BuildParams(0.01, 0.08)
    holder = {}

    def build():
        holder["t"] = None
        holder["t"] = P.construct(filtered_d, params, device=dev.index)

    b_med, b_min = timed(build)
    filtered = filtered_d.cpu().numpy()
    pre = {"raw_points": int(len(raw)), "filtered_points": int(len(filtered)),
           "filter_ms": f_med, "filter_ms_min": f_min, "build_ms": b_med, "build_ms_min": b_min,
           "timing": f"wall clock per call incl. synchronisation, median of {reps} after a "
                     "warm-up; device-resident input; build = CAPT + clearance field",
           "paper_cpu_1core_ms": {"filter": PAPER_FILTER_MS, "build": PAPER_BUILD_MS,
                                  "frame_points": 307200,
                                  "source": "ref PAPER.md:766-770 (VAMP C++, one core)"}}
    if cpu:
        from oracle import oracle as O
        t0 = time.perf_counter()
        ref_f = O.filter_cloud(raw, r_f)
        pre["filter_cpu_port_ms"] = (time.perf_counter() - t0) * 1e3
        t0 = time.perf_counter()
        O.construct(ref_f, 0.01, 0.08)
        pre["build_cpu_port_ms"] = (time.perf_counter() - t0) * 1e3
        pre["cpu_port"] = (f"oracle/capt_oracle.c filter_cloud (1 thread) and construct "
                           f"(OpenMP x{cpu_threads()}) on {cpu_model()}")
        pre["filtered_cloud_bit_exact"] = bool(
            ref_f.shape == filtered.shape and
            np.array_equal(ref_f.view(np.uint32), filtered.view(np.uint32)))
    return filtered, holder["t"], pre


# --------------------------------------------------------------------------
# main (our arm)
# --------------------------------------------------------------------------

def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return main_reference(args, rank, world)
    if args.sweep:
        return main_sweep(args)

    import torch
    import torch.distributed as dist
    import paper_2406_02807_b200 as P
    from paper_2406_02807_b200 import _lib
    from paper_2406_02807_b200.dist import reduce_counters, replicate_tree, shard_range

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    spec = W.CONFIGS[args.config]
    L = spec.lane_width
    lib = _lib.lib()

    # ---- tree (and for config 2 the timed preprocessing) on rank 0,
    #      replicated by one NCCL broadcast of the slab
    tree, build_ms, pre = None, None, None
    cloud = None
    if args.config == 2:
        cloud, tree0, pre = preprocess_cfg2(P, dev, cpu=(rank == 0 and not args.no_parity))
        if rank == 0:
            tree = tree0
        build_ms = pre["build_ms"]
    else:
        cloud = cloud_for(args.config)
        if rank == 0:
            # (a first build warms the allocator and the kernels; the best of
            # two more is reported -- the slab's cudaMalloc varies run to run)
            params = P.BuildParams(spec.r_min, spec.r_max)
            tree = P.construct(P.PointCloud(cloud), params, device=local)
            times = []
            for _ in range(2):
                tree = None
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                tree = P.construct(P.PointCloud(cloud), params, device=local)
                torch.cuda.synchronize()
                times.append((time.perf_counter() - t0) * 1e3)
            build_ms = min(times)
    if world > 1:
        tree = replicate_tree(tree, src=0, device=local)

    # ---- this rank's queries
    if args.scaling == "strong":
        c_all, r_all = batch_for(args.config, 0, cloud)
        s0, s1 = shard_range(len(r_all) // L, world, rank, align=32)
        c_np, r_np = c_all[s0 * L: s1 * L], r_all[s0 * L: s1 * L]
    else:
        c_all = r_all = None
        c_np, r_np = batch_for(args.config, rank, cloud)
    n = len(r_np)
    mode = {"auto": 0, "direct": _lib.MODE_DIRECT, "binned": _lib.MODE_BINNED}[args.mode]
    c_d = torch.from_numpy(np.ascontiguousarray(c_np)).to(dev)
    r_d = torch.from_numpy(np.ascontiguousarray(r_np)).to(dev)
    ng = n // L
    words = torch.zeros(max((ng + 31) // 32, 1), dtype=torch.int32, device=dev)
    bad = torch.full((1,), -1, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        P.query_bits(tree, c_d, r_d, L, out=words, first_bad=bad, check_radii=True,
                     mode=mode, stream=stream.cuda_stream)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if int(bad.item()) >= 0:
        raise ValueError("radius outside the band in the synthetic workload")
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = lib.capt_kernel_launches()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    launches = lib.capt_kernel_launches() - launches0
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    t_ms = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
    ms_max = float(t_ms.item())
    ms_per_step = ms_max / args.steps
    n_job = n * world if args.scaling == "weak" else len(r_all)
    value = n_job * args.steps / (ms_max * 1e-3)
    words_host = words.cpu().numpy().copy()

    # ---- per-stage split from CUDA events capt_query records around its
    # kernels on `stream`, over a second run of the same K steps (events
    # between the kernels would cost the timed steps their programmatic
    # launch overlap)
    lib.capt_stage_timing(1)
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    st_ms = (ctypes.c_double * 3)()
    st_calls = ctypes.c_int64(0)
    _lib.check(lib.capt_stage_times(st_ms, ctypes.byref(st_calls)))
    lib.capt_stage_timing(0)
    lc = (ctypes.c_uint32 * 3)()
    have_lists = lib.capt_field_list_counts(ctypes.c_void_p(stream.cuda_stream), lc) == 0

    # ---- reference counters of the same batch from the device counter
    # kernel (CAPT_STATS: collisions, boundary spheres, counted tests), then
    # the one collective of the query path: the count all-reduce
    counters = torch.zeros(6, dtype=torch.int64, device=dev)
    P.query_bits(tree, c_d, r_d, L, out=torch.empty_like(words), counters=counters, mode=mode,
                 stream=stream.cuda_stream)
    torch.cuda.synchronize()
    tot = reduce_counters(counters).cpu().numpy().astype(np.int64)

    # ---- roofline
    hbm_peak, peak_src = 6546.2, "fallback"
    mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        hbm_peak, peak_src = float(json.load(open(mp)).get("hbm_gbs", hbm_peak)), \
            "MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth)"
    peak_fp32 = ctypes.c_double(0.0)
    _lib.check(lib.capt_measure_fp32_peak(local, ctypes.byref(peak_fp32)))
    bytes_step = 16 * n + 4 * words.numel()  # sphere stream in, verdict words out
    calls = int(st_calls.value)
    roof = None
    if calls == args.steps:
        k0_ms, list_ms = st_ms[0] / calls, st_ms[1] / calls
        k0_name = "k_resolve1" if L in (1, 4, 8, 16) else "k_resolve<"
        roof = {"bound": "hbm", "kernel": f"{k0_name.rstrip('<')} (K0: clearance-field resolve)",
                "achieved": bytes_step / (k0_ms * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s"}
        roof["frac"] = roof["achieved"] / roof["peak"]
        roof["traffic"], roof["traffic_source"] = profiled_traffic(args.config, k0_name)
        roof["algorithmic_bytes_per_launch"] = bytes_step
        roof["algorithmic_bytes_definition"] = ("16 B per sphere (fp32 x, y, z, r) + the verdict "
                                                "words (SURVEY 8d); the L2-resident field records "
                                                "K0 gathers are not HBM traffic")
        roof["kernel_ms"] = k0_ms
        stages = [{"kernel": roof["kernel"], "ms": k0_ms, "share_of_step": k0_ms / ms_per_step,
                   "bound": "hbm", "algorithmic_bytes": bytes_step,
                   "achieved_gbs": roof["achieved"], "frac": roof["frac"]}]
        if have_lists:
            n1, n2, n3 = int(lc[0]), int(lc[1]), int(lc[2])
            mean_set = float(tree.stats().mean_affordance)
            lbytes = n1 * (20 + 20 + CAND_RECORD_BYTES) + (n2 + n3) * 20 + \
                n3 * 12 * mean_set
            stages.append({
                "kernel": "k_list_knn + k_bucket_list + k_tree_list (list stage)", "ms": list_ms,
                "share_of_step": list_ms / ms_per_step, "bound": "hbm",
                "entries": n1, "entries_bucket_scan": n2, "entries_tree_path": n3,
                "algorithmic_bytes": lbytes,
                "algorithmic_bytes_definition": "per entry: 20 B written by K0 + read back, "
                                                "a 192-B candidate record; per bucket-scan or "
                                                "tree-path entry its sphere; per tree-path entry "
                                                "the mean affordance set (12 B/pt)",
                "achieved_gbs": lbytes / (list_ms * 1e-3) / 1e9,
                "frac": lbytes / (list_ms * 1e-3) / 1e9 / hbm_peak,
                "note": "latency-bound: a few thousand dependent record gathers per step"})
        roof["stages"] = stages
    else:  # forced tree-only pipelines: the whole step against the HBM stream
        roof = {"bound": "hbm", "kernel": f"whole step ({args.mode} pipeline)",
                "achieved": bytes_step / (ms_per_step * 1e-3) / 1e9, "peak": hbm_peak,
                "unit": "GB/s", "traffic": None, "algorithmic_bytes_per_launch": bytes_step}
        roof["frac"] = roof["achieved"] / roof["peak"]
    roof["peak_source"] = peak_src
    tests = int(tot[2])
    roof["reference_work"] = {
        "definition": "SURVEY 8d's bound on the reference's own work: max(streamed bytes / HBM "
                      "peak, 8 flop x the reference's counted distance tests / FP32 peak) vs the "
                      "step.  The clearance field decides most spheres without any distance test, "
                      "so this is the work the product avoids, not a bound on its kernels",
        "counted_tests_per_step": tests,
        "fp32_peak_tflops": peak_fp32.value,
        "reference_work_ms": max(bytes_step / (hbm_peak * 1e9),
                                 FLOP_PER_TEST * tests / (peak_fp32.value * 1e12)) * 1e3,
        "speedup_over_reference_work_at_peak":
            max(bytes_step / (hbm_peak * 1e9),
                FLOP_PER_TEST * tests / (peak_fp32.value * 1e12)) * 1e3 / ms_per_step}

    # ---- parity: the whole job's verdict words on rank 0 vs the oracle
    parity = None
    if not args.no_parity:
        all_words = [words_host]
        if world > 1:
            cnt = torch.tensor([words.numel()], dtype=torch.int64, device=dev)
            sizes = [torch.zeros_like(cnt) for _ in range(world)]
            dist.all_gather(sizes, cnt)
            mx = int(max(s.item() for s in sizes))
            buf = torch.zeros(mx, dtype=torch.int32, device=dev)
            buf[: words.numel()] = words
            gath = [torch.zeros_like(buf) for _ in range(world)]
            dist.all_gather(gath, buf)
            all_words = [g[: int(s.item())].cpu().numpy() for g, s in zip(gath, sizes)]
        if rank == 0:
            parity = run_parity(args, tree, cloud, c_np, r_np, c_all, r_all, all_words, world, L,
                                pre, int(tot[1]))
        if world > 1:
            dist.barrier()

    # ---- e2e: the C-ABI call a plugin makes (capt_query with CAPT_HOST_IO)
    # on pinned fp32 host buffers -- H2D of the spheres, the kernels and the
    # D2H of the verdict words inside the region; beside it the reference
    # caller's path: collides_many on pageable float64 numpy arrays
    e2e = None
    if args.e2e_steps > 0:
        from paper_2406_02807_b200.query import collides_many as py_collides_many
        c_pin = torch.from_numpy(np.ascontiguousarray(c_np)).pin_memory().numpy()
        r_pin = torch.from_numpy(np.ascontiguousarray(r_np)).pin_memory().numpy()
        n_words = (ng + 31) // 32
        w_pin = torch.zeros(n_words, dtype=torch.int32).pin_memory().numpy().view(np.uint32)
        fb = ctypes.c_int64(-1)
        flags = _lib.HOST_IO | _lib.PREFILTER | _lib.CHECK_RADII | mode

        def abi_call():
            _lib.check(lib.capt_query(tree.handle, c_pin.ctypes.data, r_pin.ctypes.data, n, L,
                                      None, flags, w_pin.ctypes.data, None, ctypes.byref(fb),
                                      None), "capt_query")

        abi_call()
        if world > 1:
            dist.barrier()
        # (every call timed on its own; the median call, as the reference's
        # own protocol takes a median -- a host hiccup in one of a few calls
        # would otherwise set the figure)
        ts = []
        for _ in range(args.e2e_steps):
            t0 = time.perf_counter()
            abi_call()
            ts.append(time.perf_counter() - t0)
        dt = float(np.median(ts)) * args.e2e_steps
        assert np.array_equal(w_pin[: n_words], words_host.view(np.uint32)[: n_words])
        f64, dt64 = {}, 0.0
        if L == 1:
            c64, r64 = c_np.astype(np.float64), r_np.astype(np.float64)
            py_collides_many(tree, c64, r64)
            ts64 = []
            for _ in range(args.e2e_steps):
                t1 = time.perf_counter()
                v = py_collides_many(tree, c64, r64)
                ts64.append(time.perf_counter() - t1)
            dt64 = float(np.median(ts64)) * args.e2e_steps
            assert int(v.sum()) == int(np.unpackbits(w_pin.view(np.uint8)).sum())
            f64 = {"f64_pageable_api": "paper_2406_02807_b200.collides_many(tree, float64 numpy "
                                       "centers, float64 numpy radii) -> numpy bool, the reference "
                                       "caller's path (ref query.py:184-193)",
                   "f64_h2d_bytes_per_step": int(c64.nbytes + r64.nbytes)}
        t_e = torch.tensor([dt, dt64], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t_e, op=dist.ReduceOp.MAX)
        dt, dt64 = float(t_e[0].item()), float(t_e[1].item())
        if f64:
            f64["f64_pageable_value"] = n_job * args.e2e_steps / dt64
        e2e = {"value": n_job * args.e2e_steps / dt,
               "unit": UNIT, "h2d_bytes_per_step": int(c_pin.nbytes + r_pin.nbytes),
               "d2h_bytes_per_step": int(n_words * 4),
               "api": "capt_query(CAPT_HOST_IO) C-ABI, pinned fp32 host buffers in, verdict "
                      "words out (per rank)",
               "timing": f"median of {args.e2e_steps} calls after one warm-up call, wall clock "
                         "around each call (the call returns with the words on the host)",
               **f64}

    # ---- CPU baselines (rank 0 at N = 1 only)
    cpu_base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O
        ref_tree = parity.pop("_ref_tree", None) if parity else None
        if ref_tree is None:
            ref_tree = O.tree_from(tree)
        th = cpu_threads()
        rate, ns, med = cpu_port_rate(ref_tree, c_np, r_np, L, th, target_s=3.0)
        rate1, ns1, med1 = cpu_port_rate(ref_tree, c_np, r_np, L, 1, target_s=1.5)
        cpu_base = {"value": rate, "unit": UNIT, "cores": th, "kind": "port",
                    "sample": f"first {ns} spheres of the batch, oracle/capt_oracle.c OpenMP "
                              f"x{th} on {cpu_model()}, 1 warm-up + median of 3 ({med:.2f} s)",
                    "one_thread": {"value": rate1, "unit": UNIT, "cores": 1, "kind": "port",
                                   "sample": f"first {ns1} spheres, 1 warm-up + median of 3 "
                                             f"({med1:.2f} s)"}}
        pyref = python_reference_rate(tree, c_np, r_np, L, target_s=1.5)
        if pyref is not None:
            cpu_base["python_reference"] = pyref
    if parity:
        parity.pop("_ref_tree", None)

    if rank == 0:
        st = tree.stats()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (seeded generators, paper_2406_02807_b200/workloads.py)",
            "config": config_block(args, world),
            "groups_per_s": value / L if L > 1 else None,
            "tree": {"leaves": tree.n, "stored_points": int(st.total_stored),
                     "max_affordance": int(st.max_affordance),
                     "mean_affordance": float(st.mean_affordance),
                     "device_bytes": int(tree.device_bytes), "build_ms_rank0": build_ms,
                     "build_timing": "wall clock of construct (tree + clearance field), host "
                                     "cloud in: best of 2 after a warm-up build"},
            "preprocess": pre,
            "counters": {"collisions": int(tot[0]), "boundary_spheres": int(tot[1]),
                         "counted_tests": int(tot[2]), "fixups": int(tot[3]),
                         "aabb_rejections": int(tot[4]),
                         "source": "device counter kernel (CAPT_STATS), summed over ranks"},
            "parity": parity,
            "roofline": roof, "cpu_baseline": cpu_base, "e2e": e2e,
            "gpu_launches": int(launches), "clocks": clk.summary(),
        }
        print(json.dumps(line))
        if parity and parity.get("mismatches"):
            print(f"PARITY FAILURE: {parity}", file=sys.stderr)
            sys.exit(3)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_parity(args, tree, cloud, c_np, r_np, c_all, r_all, all_words, world, L, pre,
               dev_boundary):
    """Rank 0: the device tree vs the oracle's construct of the same cloud,
    then every rank's verdict words vs the oracle (OpenMP, every host
    thread) on that tree."""
    from oracle import oracle as O
    from oracle.parity import mask_parity, tree_parity
    spec = W.CONFIGS[args.config]
    th = cpu_threads()
    t0 = time.perf_counter()
    tp = tree_parity(tree, cloud, spec.r_min, spec.r_max)
    ref_tree = tp.pop("ref")
    t_tree = time.perf_counter() - t0
    t0 = time.perf_counter()
    if args.scaling == "strong":
        words = np.concatenate([w.view(np.uint32) for w in all_words])
        batches = [(c_all, r_all, words)]
    else:
        batches = [(c_np, r_np, all_words[0])]
        # the other ranks' batches are regenerated from their seeds (bounded)
        for rk in range(1, world):
            if (rk + 1) * len(r_np) > (1 << 28):
                break
            cr, rr = batch_for(args.config, rk, cloud)
            batches.append((cr, rr, all_words[rk]))
    res = {"spheres": 0, "units": 0, "mismatches": 0, "collisions": 0, "boundary": 0}
    for c, r, w in batches:
        m = mask_parity(ref_tree, c, r, w, L, threads=th)
        for k in res:
            res[k] += m[k]
    t_mask = time.perf_counter() - t0
    out = {"spheres": res["spheres"], "units": res["units"],
           "unit": "groups of 8 (any-collision bits)" if L > 1 else "spheres",
           "mismatches": res["mismatches"], "collisions": res["collisions"],
           "boundary": res["boundary"], "boundary_device_counter_rank_sum": dev_boundary,
           "boundary_definition": "spheres with some affordance-set point of their leaf at "
                                  "|d^2 - r^2| < 1e-6 (float64; SURVEY 8c), counted by the "
                                  "oracle over every sphere",
           "ranks_checked": len(batches) if args.scaling == "weak" else world,
           "tree": {k: v for k, v in tp.items()},
           "oracle": f"oracle/capt_oracle.c construct + collides_{'groups' if L > 1 else 'many'}"
                     f", OpenMP x{th}; tree {t_tree:.1f} s, masks {t_mask:.1f} s",
           "_ref_tree": ref_tree}
    if pre is not None and "filtered_cloud_bit_exact" in pre:
        out["filtered_cloud_bit_exact"] = pre["filtered_cloud_bit_exact"]
        if not pre["filtered_cloud_bit_exact"]:
            out["mismatches"] += 1
    out["mismatches"] += int(tp["mismatches"])
    return out


# --------------------------------------------------------------------------
# config 4 sweep
# --------------------------------------------------------------------------

def main_sweep(args):
    """Config 4 (BASELINE.json configs[4]): batch size (4^5 .. 4^14 spheres)
    x collision rate (0, 10, 50, 90, 100 %) on the config-1 cloud, per-sphere
    verdicts.  Each rate's spheres come from a 4M-sphere labelled pool
    (colliding / rejection-sampled free centres, workloads.cfg4_queries)
    tiled to the batch size; the pool's device verdicts are compared with the
    oracle (and the generator's labels), the achieved collision rate is the
    oracle's.  Prints one JSON object with the grid."""
    import torch
    import paper_2406_02807_b200 as P
    from paper_2406_02807_b200 import _lib
    from oracle import oracle as O
    from oracle.parity import unpack_words

    dev = torch.device("cuda", 0)
    cloud = W.cfg1_cloud()
    tree = P.construct(P.PointCloud(cloud), P.BuildParams(0.02, 0.08), device=0)
    ref_tree = O.construct(cloud, 0.02, 0.08)
    pool_n = 1 << 22
    mflag = {"auto": 0, "direct": _lib.MODE_DIRECT, "binned": _lib.MODE_BINNED}[args.mode]
    rows, checks = [], []
    stream = torch.cuda.current_stream(dev)
    for rate in (0.0, 0.1, 0.5, 0.9, 1.0):
        c, r, label = W.cfg4_queries(cloud, pool_n, rate, seed=104)
        cd, rd = torch.from_numpy(c).to(dev), torch.from_numpy(r).to(dev)
        words = P.query_bits(tree, cd, rd, 1, check_radii=False)
        got = unpack_words(words.cpu().numpy(), pool_n)
        exp = O.collides_many(ref_tree, c, r, threads=cpu_threads())
        checks.append({"rate": rate, "pool": pool_n, "mismatches": int((got != exp).sum()),
                       "oracle_rate": float(exp.mean()),
                       "labels_match": bool(np.array_equal(exp, label))})
        for e in range(5, args.sweep_max_exp + 1):
            n = 4 ** e
            reps = -(-n // pool_n)
            cN = cd.repeat(reps, 1)[:n].contiguous() if reps > 1 else cd[:n].contiguous()
            rN = rd.repeat(reps)[:n].contiguous() if reps > 1 else rd[:n].contiguous()
            out = torch.empty((n + 31) // 32, dtype=torch.int32, device=dev)

            def q(s=stream):
                P.query_bits(tree, cN, rN, 1, out=out, check_radii=False,
                             stream=s.cuda_stream, mode=mflag)

            for _ in range(3):
                q()
            steps = max(3, min(200, int(2e8 // n)))
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(steps):
                q()
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / steps
            # tiled pools: every copy's verdicts equal the pool's
            wn = out.cpu().numpy()
            ok = bool(np.array_equal(unpack_words(wn, n), np.tile(got, reps)[:n]))
            rows.append({"rate": rate, "n": n, "ms": ms, "queries_per_s": n / (ms * 1e-3),
                         "mode": args.mode if args.mode != "auto" else
                         ("field" if n >= 8192 else "warp"), "tiled_verdicts_match": ok})
            del cN, rN, out
    print(json.dumps({"sweep": "cfg4 batch size x collision rate", "n_gpus": 1,
                      "tree_leaves": tree.n, "pool": pool_n, "oracle_checks": checks,
                      "rows": rows}))


# --------------------------------------------------------------------------
# reference arm
# --------------------------------------------------------------------------

def main_reference(args, rank, world):
    """The reference algorithm on the host CPU: the oracle port
    (oracle/capt_oracle.c, a restatement of captree's construct and
    collides_many / collides_batch) over every host thread, on each step a
    bounded prefix of the same batch.  Rank 0 alone runs and prints."""
    if rank != 0:
        return
    from oracle import oracle as O
    spec = W.CONFIGS[args.config]
    L = spec.lane_width
    if args.config == 2:
        cloud = O.filter_cloud(W.cfg2_raw_cloud(), 0.01)
    else:
        cloud = cloud_for(args.config)
    tree = O.construct(cloud, spec.r_min, spec.r_max)
    c, r = batch_for(args.config, 0, cloud)
    threads = cpu_threads()
    c64, r64 = c.astype(np.float64), r.astype(np.float64)
    # each step ~min(2 s, 60 s / (K + W)) of CPU work
    per_step_s = min(2.0, 60.0 / max(1, args.steps + args.warmup))
    per_step = size_sample(lambda m: _oracle_run(O, tree, c64[:m], r64[:m], L, threads), L,
                           per_step_s, len(r))
    cc, rr = c64[:per_step], r64[:per_step]
    for _ in range(args.warmup):
        _oracle_run(O, tree, cc, rr, L, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        _oracle_run(O, tree, cc, rr, L, threads)
    dt = time.perf_counter() - t0
    value = per_step * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generators, paper_2406_02807_b200/workloads.py)",
        "config": config_block(args, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"first {per_step} spheres of the batch per step, "
                                   f"oracle/capt_oracle.c OpenMP x{threads} on {cpu_model()}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
