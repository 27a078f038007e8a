"""Turn gpurun ncu outputs into the committed profile summaries.

    python profiles/summarize.py launches <launches.csv> <out.md>
    python profiles/summarize.py full <report.ncu-rep> <out.json>
    python profiles/summarize.py sweep <sweep.json> <out.md>

``launches``: per-kernel device time from an
``ncu --metrics gpu__time_duration.sum --clock-control none`` launch list
(cold-cache, serialised: compare shares, not absolutes).
``full``: headline metrics of every kernel in an ``ncu --set full`` report
(duration, DRAM bytes, throughputs, IPC, occupancy, FP32/FMA pipe use).
"""

from __future__ import annotations

import collections
import csv
import json
import subprocess
import sys


def launches(path: str, out: str) -> None:
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("capt::", "").replace("<unnamed>::", "")
        agg.setdefault(name, []).append(float(d["Metric Value"]) / 1e3)
    lines = [f"# Kernel launch list: {path.split('/')[-1]}", "",
             "| kernel | launches | mean us | total us |", "|---|---:|---:|---:|"]
    for k, v in agg.items():
        lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.1f} | {sum(v):.1f} |")
    open(out, "w").write("\n".join(lines) + "\n")


WANT = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "lts__t_sector_hit_rate.pct": "l2_hit_rate_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__inst_executed.avg.per_cycle_active": "ipc_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_inst_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "smsp__inst_executed.sum": "warp_instructions",
}


def full(path: str, out: str) -> None:
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        item = {"kernel": d.get("Kernel Name", "")[:120]}
        for k, name in WANT.items():
            if k in d:
                item[name] = d[k]
                if u.get(k):
                    item[name + "_unit"] = u[k]
        res.append(item)
    json.dump(res, open(out, "w"), indent=1)


def sweep(path: str, out: str) -> None:
    """bench.py --sweep JSON line -> markdown table (G sphere queries/s per
    call | with CUDA-graph replay, path taken, label check)."""
    d = json.loads(open(path).read().strip().splitlines()[-1])
    rows = d["rows"]
    rates = sorted({r["rate"] for r in rows})
    ns = sorted({r["n"] for r in rows})
    lines = [f"# {d['sweep']} (1x B200, tree {d['tree_leaves']} leaves)", "",
             "G sphere queries/s: per call | CUDA-graph replay; path f = clearance field "
             "(default), d = unbinned tree kernels, b = binned; ! = label mismatch", "",
             "| spheres | " + " | ".join(f"rate {x}" for x in rates) + " |",
             "|---:|" + "---:|" * len(rates)]
    for n in ns:
        cells = []
        for x in rates:
            r = [q for q in rows if q["n"] == n and q["rate"] == x][0]
            cells.append(f"{r['queries_per_s'] / 1e9:.2f} \\| {r['queries_per_s_graph'] / 1e9:.2f} "
                         f"{r['mode'][0]}{'' if r['labels_match'] else ' !'}")
        lines.append(f"| {n:,} | " + " | ".join(cells) + " |")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    {"launches": launches, "full": full, "sweep": sweep}[sys.argv[1]](sys.argv[2], sys.argv[3])
