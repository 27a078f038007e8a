"""Benchmark: CAPT batched sphere-collision queries on B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

Default workload = BASELINE.json configs[1]: the tabletop box scene (16,384
points, CAPT r_min 0.02 / r_max 0.08) queried with 4,194,304 spatially
correlated groups of 8 spheres per GPU (33,554,432 sphere queries), one
any-collision bit per group (edge-validation early-exit semantics,
query.py:126-167).  Multi-GPU (torchrun): the tree is built on rank 0 and
replicated by an NCCL broadcast of its device slab; every rank queries its own
4M groups (weak scaling, no data-path collective); the counters are summed
with one NCCL all-reduce at the end.

One "step" = one capt_query over the rank's whole batch with inputs resident
in HBM (512 MB of spheres per step > the 126 MB L2, so no flush is needed).
``e2e`` times the same batch through the public API with host (pinned)
buffers, the host->device copy of the spheres and the device->host copy of
the verdict bits inside the timed region.

``--impl reference`` times the reference algorithm on the host CPU: the
oracle port (oracle/capt_oracle.c, a restatement of captree.collides_batch /
collides_many) with every host thread, on a bounded sample of the same
workload per step.  Rank 0 alone runs it.
"""

from __future__ import annotations

import argparse
import json
import os
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=1, choices=[0, 1, 3])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="auto", choices=["auto", "direct", "binned"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sweep", action="store_true",
                    help="config-4 batch-size x collision-rate sweep (one JSON object)")
    ap.add_argument("--sweep-max-exp", type=int, default=13,
                    help="largest batch is 4^this spheres (14 -> 268M, needs ~4.3 GB)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# --------------------------------------------------------------------------
# workloads
# --------------------------------------------------------------------------

def workload(cfg: int, rank: int, scale: float = 1.0):
    """(cloud, r_min, r_max, centers, radii, lane_width, description)."""
    spec = W.CONFIGS[cfg]
    if cfg == 0:
        cloud = W.cfg0_cloud()
        n = int(spec.n_queries * scale)
        c, r = W.cfg0_queries(n, seed=1 + 1000 * rank)
        desc = "cfg0: 2,048 uniform points, 1,048,576 independent spheres per GPU"
    elif cfg == 1:
        cloud = W.cfg1_cloud()
        g = int((spec.n_queries // 8) * scale)
        c, r = W.cfg1_queries(cloud, n_groups=g, seed=101 + 1000 * rank)
        desc = ("cfg1: tabletop scene (16,384 pts), 4,194,304 groups x 8 spheres per GPU, "
                "one any-collision bit per group")
    else:
        cloud = W.cfg3_cloud()
        n = int(spec.n_queries * scale)
        c, r = W.cfg3_queries(n, seed=103 + 1000 * rank)
        desc = "cfg3: 262,144-pt Gaussian mixture, 67,108,864 spheres per GPU"
    return cloud, spec.r_min, spec.r_max, c, r, spec.lane_width, desc


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
# CPU reference (oracle port, all host threads)
# --------------------------------------------------------------------------

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


def profiled_traffic(config, name="ncu_full", only=None):
    """DRAM bytes (read + write) per launch from the committed ncu --set full
    capture of this bench command (profiles/r01_cfg<k>_<name>.json, summed
    over the captured kernels whose name contains ``only``), or (None, why)."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                        f"r01_cfg{config}_{name}.json")
    if not os.path.exists(path):
        return None, "no ncu capture committed for this config"
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    total, names = 0.0, []
    for k in json.load(open(path)):
        if only and only not in k["kernel"]:
            continue
        for f in ("dram_read", "dram_write"):
            total += float(k[f]) * scale.get(k.get(f + "_unit", "byte"), 1)
        names.append(k["kernel"].split("(")[0].split("::")[-1])
    if not names:
        return None, f"no {only} launch in {os.path.basename(path)}"
    return total, (f"{os.path.relpath(path, os.path.dirname(path) + '/..')}: dram read+write of "
                   f"{', '.join(names)} (one launch each)")


def cpu_reference_rate(tree_ref, c, r, lane_width, target_s=10.0, max_spheres=None):
    """Spheres/s of the oracle port on a bounded sample sized for ~target_s."""
    from oracle import oracle as O
    threads = cpu_threads()

    def run(n):
        n -= n % lane_width
        cc, rr = c[:n].astype(np.float64), r[:n].astype(np.float64)
        t0 = time.perf_counter()
        if lane_width > 1:
            O.collides_groups(tree_ref, cc, rr, lane_width, threads=threads)
        else:
            O.collides_many(tree_ref, cc, rr, threads=threads)
        return n, time.perf_counter() - t0

    n, dt = run(min(len(r), 1 << 17))
    rate = n / max(dt, 1e-9)
    n = int(min(len(r), max_spheres or len(r), rate * target_s))
    n, dt = run(max(n, lane_width))
    # the whole batch finishes in well under target_s: repeat passes over it
    passes = 1
    if dt < 0.5 * target_s and max_spheres is None:
        passes = max(1, int(target_s / max(dt, 1e-9)))
        t0 = time.perf_counter()
        for _ in range(passes):
            run(n)
        dt = time.perf_counter() - t0
    return n * passes / dt, n, dt, threads, passes


# --------------------------------------------------------------------------
# main
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

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    cloud, r_min, r_max, c_np, r_np, L, desc = workload(args.config, rank)
    n = len(r_np)
    params = P.BuildParams(r_min, r_max)

    # tree: built on rank 0, replicated by an NCCL broadcast of its device slab
    from paper_2406_02807_b200.dist import reduce_counters, replicate_tree
    tree, build_ms = None, None
    if rank == 0:
        t0 = time.perf_counter()
        tree = P.construct(P.PointCloud(cloud), params, device=local)
        torch.cuda.synchronize()
        build_ms = (time.perf_counter() - t0) * 1e3
    if world > 1:
        tree = replicate_tree(tree, src=0, device=local)

    mode = {"auto": 0, "direct": _lib.MODE_DIRECT, "binned": _lib.MODE_BINNED}[args.mode]
    c_d = torch.from_numpy(c_np).to(dev)
    r_d = torch.from_numpy(r_np).to(dev)
    ng = n // L
    words = torch.empty((ng + 31) // 32, dtype=torch.int32, device=dev)
    bad = torch.full((1,), -1, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        P.query_bits(tree, c_d, r_d, L, out=words, first_bad=bad, check_radii=True,
                     mode=mode, stream=stream.cuda_stream)

    # counted distance tests (reference points_scanned semantics) for the roofline
    counters = torch.zeros(6, dtype=torch.int64, device=dev)
    P.query_bits(tree, c_d, r_d, L, out=words, counters=counters, mode=mode,
                 stream=stream.cuda_stream)
    torch.cuda.synchronize()
    cnt = counters.cpu().numpy().astype(np.int64)
    if int(bad.item()) >= 0:
        raise ValueError("radius outside the band in the synthetic workload")
    hits_ref = int(cnt[0])

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.lib().capt_kernel_launches()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    import ctypes
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    launches = _lib.lib().capt_kernel_launches() - launches0
    # the per-stage split (K0 / list stage) from CUDA events that capt_query
    # records around its kernels on `stream`, over a second run of the same
    # K steps (the events sit between the kernels and would cost the timed
    # steps their programmatic-launch overlap, ~9 us per config-1 step)
    _lib.lib().capt_stage_timing(1)
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    st_ms = (ctypes.c_double * 3)()
    st_calls = ctypes.c_int64(0)
    _lib.check(_lib.lib().capt_stage_times(st_ms, ctypes.byref(st_calls)))
    _lib.lib().capt_stage_timing(0)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    t_ms = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
    ms_max = float(t_ms.item())
    ms_per_step = ms_max / args.steps

    # final count reduction over NCCL (the only collective of the query path)
    tot = reduce_counters(counters.clone()).cpu().numpy().astype(np.int64)

    value = world * n * args.steps / (ms_max * 1e-3)

    # roofline.  The survey's definition is the slower of the
    # streamed bytes at HBM peak and 8 flop x the reference's counted distance
    # tests at FP32 peak, against the step time.  The product resolves most
    # spheres without any distance test (clearance field), so its dominant
    # kernel K0 is bound by the sphere stream: the primary roofline is K0's
    # algorithmic bytes (16 B/sphere in, the verdict words out) over its
    # event-timed duration against HBM peak.
    peak_fp32 = ctypes.c_double(0.0)
    _lib.check(_lib.lib().capt_measure_fp32_peak(local, ctypes.byref(peak_fp32)))
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    tests = int(cnt[2])
    bytes_step = 16 * n + 4 * words.numel()
    flops_step = FLOP_PER_TEST * tests
    t_hbm = bytes_step / (hbm_peak * 1e9)
    t_fp32 = flops_step / (peak_fp32.value * 1e12)
    survey = {"definition": "max(streamed bytes / HBM peak, 8 flop x counted tests / FP32 peak) "
                            "over the whole step (SURVEY 8d)",
              "roofline_ms": max(t_hbm, t_fp32) * 1e3,
              "frac": max(t_hbm, t_fp32) * 1e3 / ms_per_step,
              "bound": "fp32" if t_fp32 >= t_hbm else "hbm",
              "achieved_tflops": flops_step / (ms_per_step * 1e-3) / 1e12,
              "fp32_peak_tflops": peak_fp32.value,
              "counted_tests_per_step": tests, "streamed_bytes_per_step": bytes_step}
    calls = int(st_calls.value)
    if calls == args.steps:
        k0_ms, list_ms = st_ms[0] / calls, st_ms[1] / calls
        roof = {"bound": "hbm", "kernel": "k_resolve (K0: clearance-field resolve)",
                "achieved": bytes_step / (k0_ms * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s"}
        roof["frac"] = roof["achieved"] / roof["peak"]
        roof["traffic"], roof["traffic_source"] = profiled_traffic(args.config, "field_ncu_full",
                                                                   "k_resolve<")
        roof["algorithmic_bytes_per_launch"] = bytes_step
        roof["kernel_ms"] = k0_ms
        roof["stage_ms"] = {"k0_resolve": k0_ms, "list": list_ms}
        roof["k0_share_of_step"] = k0_ms / ms_per_step
    else:  # tree-only pipelines (forced modes): the whole step against the survey roofline
        kernel_ms = ms_per_step
        if t_fp32 >= t_hbm:
            roof = {"bound": "fp32", "achieved": flops_step / (kernel_ms * 1e-3) / 1e12,
                    "peak": peak_fp32.value, "unit": "TFLOP/s"}
        else:
            roof = {"bound": "hbm", "achieved": bytes_step / (kernel_ms * 1e-3) / 1e9,
                    "peak": hbm_peak, "unit": "GB/s"}
        roof["frac"] = roof["achieved"] / roof["peak"]
        roof["traffic"], roof["traffic_source"] = profiled_traffic(args.config)
    roof["peak_source"] = ("HBM: MEASURED_PEAKS.json hbm_gbs; FP32: FFMA microbenchmark measured "
                           "live (capt_measure_fp32_peak)")
    roof["survey_roofline"] = survey

    # e2e: the C-ABI call a plugin makes (capt_query with CAPT_HOST_IO) on
    # pinned host buffers -- H2D of the spheres, the kernels and the D2H of
    # the verdict words all inside the region; the Python API (which also
    # unpacks the words to a bool array on the host) is reported beside it
    e2e = None
    if args.e2e_steps > 0:
        import ctypes as C
        from paper_2406_02807_b200 import _lib
        from paper_2406_02807_b200.query import _host_query
        c_pin = torch.from_numpy(c_np).pin_memory().numpy()
        r_pin = torch.from_numpy(r_np).pin_memory().numpy()
        n_words = (n // L + 31) // 32
        w_pin = torch.zeros(n_words, dtype=torch.int32).pin_memory().numpy().view(np.uint32)
        bad = C.c_int64(-1)
        flags = _lib.HOST_IO | _lib.PREFILTER | _lib.CHECK_RADII | mode
        lib = _lib.lib()

        def abi_call():
            _lib.check(lib.capt_query(tree.handle, c_pin.ctypes.data, r_pin.ctypes.data, n, L,
                                      None, flags, w_pin.ctypes.data, None, C.byref(bad), None),
                       "capt_query")

        abi_call()  # warm-up
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            abi_call()
        dt = time.perf_counter() - t0
        hits_e2e = int(np.unpackbits(w_pin.view(np.uint8)).sum())
        _host_query(tree, c_pin, r_pin, 0, L, None, True, True, mode=mode)  # warm-up
        t1 = time.perf_counter()
        for _ in range(args.e2e_steps):
            bits, _, fb = _host_query(tree, c_pin, r_pin, 0, L, None, True, True, mode=mode)
        dt_py = time.perf_counter() - t1
        t_e = torch.tensor([dt, dt_py], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t_e, op=dist.ReduceOp.MAX)
        dt, dt_py = float(t_e[0].item()), float(t_e[1].item())
        assert hits_e2e == hits_ref and int(bits.sum()) == hits_ref
        e2e = {"value": world * n * args.e2e_steps / dt, "unit": UNIT,
               "h2d_bytes_per_step": int(c_pin.nbytes + r_pin.nbytes),
               "d2h_bytes_per_step": int(n_words * 4),
               "api": "capt_query(CAPT_HOST_IO) C-ABI, pinned host buffers, verdict words out",
               "python_api_value": world * n * args.e2e_steps / dt_py,
               "python_api": "query._host_query: the same call + unpack to a bool array"}

    cpu_base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O
        ref_tree = O.tree_from(tree)
        rate, ns, dt, th, passes = cpu_reference_rate(ref_tree, c_np, r_np, L, target_s=10.0)
        cpu_base = {"value": rate, "unit": UNIT, "cores": th, "kind": "port",
                    "sample": f"{passes} pass(es) over the first {ns} spheres ({ns // L} groups) "
                              f"of rank 0's batch, {dt:.1f} s, oracle/capt_oracle.c OpenMP "
                              f"x{th} on {cpu_model()}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded generators, paper_2406_02807_b200/workloads.py)",
            "config": {"workload": desc, "config_index": args.config,
                       "spheres_per_gpu": n, "lane_width": L,
                       "groups_per_s": value / L if L > 1 else None,
                       "r_min": r_min, "r_max": r_max,
                       "tree": {"leaves": tree.n, "stored_points": int(tree.stats().total_stored),
                                "max_affordance": int(tree.stats().max_affordance),
                                "build_ms_rank0": build_ms},
                       "l2": "inputs (16 B/sphere, 512 MB/step) exceed the 126 MB L2; no flush",
                       "mode": args.mode, "parallelism": f"dp{world} (query shards)",
                       "collisions_total": int(tot[0]), "fixups": int(tot[3])},
            "roofline": roof, "cpu_baseline": cpu_base, "e2e": e2e,
            "gpu_launches": int(launches), "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main_sweep(args):
    """Config 4 (BASELINE.json configs[4]): batch size (4^5 .. 4^14 spheres) x
    collision rate (0, 10, 50, 90, 100 %) on the config-1 cloud, per-sphere
    verdicts.  Each rate's spheres come from a 4M-sphere labelled pool
    (colliding / rejection-sampled free centres, workloads.cfg4_queries) tiled
    to the batch size; the pool's verdicts are checked against its labels.
    Prints one JSON object with the grid."""
    import torch
    import paper_2406_02807_b200 as P
    from paper_2406_02807_b200 import _lib

    dev = torch.device("cuda", 0)
    cloud = W.cfg1_cloud()
    tree = P.construct(P.PointCloud(cloud), P.BuildParams(0.02, 0.08), device=0)
    pool_n = 1 << 22
    max_exp = args.sweep_max_exp
    from paper_2406_02807_b200 import _lib
    mflag = {"auto": 0, "direct": _lib.MODE_DIRECT, "binned": _lib.MODE_BINNED}[args.mode]
    rows = []
    for rate in (0.0, 0.1, 0.5, 0.9, 1.0):
        c, r, label = W.cfg4_queries(cloud, pool_n, rate, seed=104)
        cd, rd = torch.from_numpy(c).to(dev), torch.from_numpy(r).to(dev)
        words = P.query_bits(tree, cd, rd, 1, check_radii=False)
        got = np.unpackbits(words.cpu().numpy().view(np.uint8), bitorder="little")[:pool_n]
        label_ok = bool(np.array_equal(got.astype(bool), label))
        for e in range(5, max_exp + 1):
            n = 4 ** e
            reps = -(-n // pool_n)
            cN = cd.repeat(reps, 1)[:n].contiguous() if reps > 1 else cd[:n].contiguous()
            rN = rd.repeat(reps)[:n].contiguous() if reps > 1 else rd[:n].contiguous()
            out = torch.empty((n + 31) // 32, dtype=torch.int32, device=dev)
            stream = torch.cuda.current_stream(dev)
            for _ in range(3):
                P.query_bits(tree, cN, rN, 1, out=out, check_radii=False,
                             stream=stream.cuda_stream, mode=mflag)
            steps = max(3, min(200, int(2e8 // n)))
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(steps):
                P.query_bits(tree, cN, rN, 1, out=out, check_radii=False,
                             stream=stream.cuda_stream, mode=mflag)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / steps
            # the same query captured once in a CUDA graph and replayed: device
            # latency without the per-call Python/ctypes dispatch
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream(dev)
            side.wait_stream(stream)
            with torch.cuda.stream(side):
                P.query_bits(tree, cN, rN, 1, out=out, check_radii=False,
                             stream=side.cuda_stream, mode=mflag)
                with torch.cuda.graph(g, stream=side):
                    P.query_bits(tree, cN, rN, 1, out=out, check_radii=False,
                                 stream=side.cuda_stream, mode=mflag)
            stream.wait_stream(side)
            for _ in range(3):
                g.replay()
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(steps):
                g.replay()
            e1.record(stream)
            torch.cuda.synchronize()
            ms_graph = e0.elapsed_time(e1) / steps
            mode = args.mode if args.mode != "auto" else ("field" if n >= 8192 else "direct")
            rows.append({"rate": rate, "n": n, "ms": ms, "queries_per_s": n / (ms * 1e-3),
                         "ms_graph": ms_graph, "queries_per_s_graph": n / (ms_graph * 1e-3),
                         "mode": mode, "labels_match": label_ok})
            del g
            del cN, rN, out
    print(json.dumps({"sweep": "cfg4 batch size x collision rate", "n_gpus": 1,
                      "tree_leaves": tree.n, "pool": pool_n, "rows": rows}))


def main_reference(args, rank, world):
    if rank != 0:
        return
    from oracle import oracle as O
    cloud, r_min, r_max, c, r, L, desc = workload(args.config, 0)
    tree = O.construct(cloud, r_min, r_max)
    threads = cpu_threads()
    # size one step to ~2 s of CPU work
    rate = cpu_reference_rate(tree, c, r, L, target_s=0.5, max_spheres=len(r))[0]
    per_step = int(max(L, min(len(r), rate * 2.0)))
    per_step -= per_step % L
    cc, rr = c[:per_step].astype(np.float64), r[:per_step].astype(np.float64)

    def step():
        if L > 1:
            O.collides_groups(tree, cc, rr, L, threads=threads)
        else:
            O.collides_many(tree, cc, rr, threads=threads)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    value = per_step * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generators, paper_2406_02807_b200/workloads.py)",
        "config": {"workload": desc, "config_index": args.config, "lane_width": L,
                   "spheres_per_step": per_step},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{per_step} spheres per step (prefix of the GPU batch), "
                                   f"oracle/capt_oracle.c OpenMP x{threads} on {cpu_model()}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
