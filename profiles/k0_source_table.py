"""Per-source-line instruction counts and stall samples of K0 from an
``ncu --set full --import-source on`` report.

    python profiles/k0_source_table.py <report.ncu-rep> <kernel regex> <out.md> [title]

Reads ``ncu --page source --print-source cuda,sass --csv`` (each SASS row
carries the CUDA line it came from) and sums per line of capt_field.cu.
"""
import collections
import csv
import subprocess
import sys

rep, kern, out = sys.argv[1:4]
title = sys.argv[4] if len(sys.argv) > 4 else kern
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
name = next((r[1] for r in rows if r and r[0] == "Function Name"), kern)
per = collections.OrderedDict()
hdr = None
cur_file = ""
done_first = False
for r in rows:
    if not r:
        continue
    if r[0] == "Function Name" and hdr is not None:
        break  # (one launch is enough: later launches repeat the table)
    if r[0] == "File Name":
        cur_file = r[1]
        continue
    if r[0] == "Line No":
        hdr = {n: i for i, n in enumerate(r)}
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
        continue
    key = (cur_file.split("/")[-1] or "capt_field.cu", int(r[0]), r[1].strip())
    d = per.setdefault(key, [0, 0, 0])
    d[0] += int(float(r[hdr["Instructions Executed"]] or 0))
    d[1] += int(float(r[hdr["# Samples"]] or 0))
    d[2] += int(float(r[hdr["stall_long_sb"]] or 0))
tot_i = sum(v[0] for v in per.values())
tot_s = sum(v[1] for v in per.values())
lines = [f"# {title}", "",
         f"`{name}`: {tot_i:,} warp instructions, {tot_s:,} stall samples "
         f"({sum(v[2] for v in per.values()):,} long-scoreboard); lines with >= 1% of either.",
         "", "| file:line | warp instr | share | stall samples | share | long-scoreboard | source |",
         "|---|---:|---:|---:|---:|---:|---|"]
for (f, ln, src), (ni, ns, nl) in sorted(per.items(), key=lambda kv: -kv[1][0]):
    if ni < 0.01 * tot_i and ns < 0.01 * tot_s:
        continue
    lines.append(f"| {f}:{ln} | {ni:,} | {100 * ni / max(tot_i, 1):.1f}% | {ns:,} | "
                 f"{100 * ns / max(tot_s, 1):.1f}% | {nl:,} | `{src[:90]}` |")
open(out, "w").write("\n".join(lines) + "\n")
print(out, tot_i, tot_s)
