"""Summarise ncu outputs into profiles/<name>.md (+ a traffic json).

usage: python scripts/ncu_summary.py --launches gpurun_out/launches.csv \
           --rep gpurun_out/prof.ncu-rep --cycle-launches 63 --name r01_... \
           [--cells 134217728]
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "l1tex__t_bytes.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
]


def launch_table(path, per_cycle):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    mi = hdr.index("Metric Name")
    gi = hdr.index("Grid Size") if "Grid Size" in hdr else None
    data = [(r[ki].split("(")[0], r[gi] if gi is not None else "",
             float(r[vi].replace(",", ""))) for r in rows[1:]
            if r[mi] == "gpu__time_duration.sum"]
    ncyc = 3
    tail = data[-per_cycle * ncyc:]
    tot, cnt = defaultdict(float), defaultdict(int)
    for n, g, v in tail:
        tot[(n, g)] += v / ncyc
        cnt[(n, g)] += 1
    s = sum(tot.values())
    out = ["| kernel | grid | launches/cycle | ns/cycle | share |",
           "|---|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append("| %s | %s | %d | %.0f | %.1f%% |" % (k[0], k[1], cnt[k] // ncyc,
                                                       v, 100 * v / s))
    out.append("| **total** | | %d | %.0f | 100%% |" % (len(tail) // ncyc, s))
    return "\n".join(out), s


def rep_table(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                d[m] = (r[i], units[i])
        recs.append(d)
    return recs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep", nargs="*", default=[])
    ap.add_argument("--cycle-launches", type=int, default=63)
    ap.add_argument("--name", required=True)
    ap.add_argument("--cells", type=int, default=512 ** 3)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    md = ["# ncu summary: %s" % a.name, "", a.note, ""]
    if a.launches:
        t, s = launch_table(a.launches, a.cycle_launches)
        md += ["## Launch list (one V-cycle, ncu `gpu__time_duration.sum`, "
               "cold-cache serialised: compare shares, not absolutes)", "", t, ""]
    traffic = None
    for rep in a.rep:
        recs = rep_table(rep)
        md += ["## `--set full` capture: %s" % os.path.basename(rep), ""]
        for d in recs:
            md.append("### %s" % d["kernel"])
            md.append("| metric | value | unit |")
            md.append("|---|---|---|")
            for m in METRICS:
                if m in d:
                    md.append("| %s | %s | %s |" % (m, d[m][0], d[m][1]))
            try:
                rd = float(d["dram__bytes_read.sum"][0].replace(",", ""))
                wr = float(d["dram__bytes_write.sum"][0].replace(",", ""))
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                rd *= scale[d["dram__bytes_read.sum"][1]]
                wr *= scale[d["dram__bytes_write.sum"][1]]
                md.append("")
                md.append("DRAM traffic per launch: %.1f MB read + %.1f MB write"
                          " = %.2f B per fine cell" % (rd / 1e6, wr / 1e6,
                                                       (rd + wr) / a.cells))
                if traffic is None and "smooth" in d["kernel"]:
                    traffic = rd + wr
            except Exception:
                pass
            md.append("")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", a.name + ".md"), "w") as fh:
        fh.write("\n".join(md) + "\n")
    if traffic is not None:
        with open(os.path.join(ROOT, "profiles", "roofline_traffic.json"), "w") as fh:
            json.dump({"kernel": "k_smooth_march", "cells": a.cells,
                       "bytes_per_launch": traffic, "source": a.name}, fh)
    print("\n".join(md))


if __name__ == "__main__":
    main()
