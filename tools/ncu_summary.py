"""Summarise ncu captures into profiles/ (tracked): per-kernel key metrics
from --set full reports and per-launch shares from a launch-list CSV."""

from __future__ import annotations

import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
]


def short(name: str) -> str:
    name = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    return name.split("(")[0]


def report(path: str) -> str:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = [f"## {path}", "", "| kernel | " + " | ".join(KEYS) + " |", "|" + "---|" * (len(KEYS) + 1)]
    for r in rows[2:]:
        cells = []
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                cells.append(f"{r[i]} {units[i]}".strip())
            else:
                cells.append("-")
        out.append(f"| {short(r[hdr.index('Kernel Name')])} | " + " | ".join(cells) + " |")
    return "\n".join(out) + "\n"


DETAIL_SECTIONS = ("GPU Speed Of Light Throughput", "Memory Workload Analysis", "Compute Workload Analysis",
                   "Scheduler Statistics", "Warp State Statistics", "Occupancy")
DETAIL_KEYS = ("Duration", "SM Frequency", "Memory Throughput", "DRAM Throughput", "L1/TEX Cache Throughput",
               "L2 Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
               "L2 Hit Rate", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
               "Achieved Occupancy", "Registers Per Thread")


def detail(path: str) -> str:
    """Speed-of-light / scheduler lines and the warp-stall breakdown
    (pc sampling) of a --set full report."""
    raw = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    out = [f"## {path} (--set full)", "", "| kernel | section | metric | value |", "|---|---|---|---|"]
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Section Name") in DETAIL_SECTIONS and d.get("Metric Name") in DETAIL_KEYS:
            out.append(f"| {short(d['Kernel Name'])} | {d['Section Name']} | {d['Metric Name']} | "
                       f"{d['Metric Value']} {d.get('Metric Unit', '')} |")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    pre = "smsp__pcsamp_warps_issue_stalled_"
    for r in rows[2:]:
        st = []
        for i, h in enumerate(hdr):
            if h.startswith(pre) and not h.endswith("_not_issued"):
                try:
                    st.append((float(r[i].replace(",", "")), h[len(pre):]))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1.0
        out += ["", f"warp-stall samples, {short(r[hdr.index('Kernel Name')])}:", "",
                "| reason | share |", "|---|---|"]
        out += [f"| {k} | {100 * v / tot:.1f}% |" for v, k in sorted(st, reverse=True)[:10]]
    return "\n".join(out) + "\n"


def launches(path: str, skip_prefix_kernels: int = 0) -> str:
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        tot[short(r[ki])] += v
        cnt[short(r[ki])] += 1
    unit = rows[1][hdr.index("Metric Unit")] if "Metric Unit" in hdr else "?"
    all_t = sum(tot.values())
    out = [f"## {path} (all launches of the command; ncu serialises, cold caches)", "",
           f"| kernel | launches | total ({unit}) | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        out.append(f"| {k} | {cnt[k]} | {v:.1f} | {100 * v / all_t:.1f}% |")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    out = sys.argv[1]
    parts = []
    for a in sys.argv[2:]:
        if a.endswith(".csv"):
            parts.append(launches(a))
        else:
            parts.append(report(a))
            parts.append(detail(a))
    open(out, "w").write("\n".join(parts))
    print(open(out).read())
