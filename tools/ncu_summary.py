"""Summarise ncu captures into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py full  gpurun_out/attn_full.ncu-rep  profiles/r01_attn_full.md
    python tools/ncu_summary.py launches gpurun_out/launches.csv   profiles/r01_launches.md

`full` extracts the roofline-relevant raw metrics (duration, DRAM bytes, tensor / XU /
FMA pipe utilisation, registers, occupancy, top warp-stall SASS lines); `launches`
aggregates the per-launch duration list (cold-cache, serialised) into per-kernel shares.
"""
from __future__ import annotations

import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict

RAW_KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warp_latency_per_inst_issued.ratio",
]


def ncu_csv(args):
    out = subprocess.run(["ncu"] + args, capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def full(rep, dest):
    rows = ncu_csv(["-i", rep, "--page", "raw", "--csv"])
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary: `{rep}`", ""]
    summary = []
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")]
        lines.append(f"## {name[:120]}")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        rec = {"kernel": name}
        for k in RAW_KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"| {k} | {vals[i]} | {units[i]} |")
                rec[k] = vals[i]
        summary.append(rec)
        lines.append("")
    # top stall locations (SASS) for the first kernel
    try:
        src = ncu_csv(["-i", rep, "--page", "source", "--csv", "--print-source", "sass"])
        h = src[1]
        data = src[2:]
        ia, isrc = h.index("Address"), h.index("Source")
        iss = h.index("Warp Stall Sampling (All Samples)")
        tot = sum(float(r[iss] or 0) for r in data) or 1.0
        lines += ["## top warp-stall SASS lines (all samples)", "", "| share | SASS |", "|---|---|"]
        for r in sorted(data, key=lambda r: -float(r[iss] or 0))[:25]:
            lines.append(f"| {float(r[iss]) / tot * 100:.1f}% | `{r[isrc].strip()[:100]}` |")
    except (subprocess.CalledProcessError, ValueError, IndexError):
        pass
    with open(dest, "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(dest.rsplit(".", 1)[0] + ".json", "w") as f:
        json.dump(summary, f, indent=1)
    print(dest)


def launches(path, dest):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[1:]:
        name = re.sub(r"\(.*", "", r[ki])[:80]
        agg[name].append(float(r[vi]))
    tot = sum(sum(v) for v in agg.values())
    lines = [f"# ncu launch list (gpu__time_duration.sum, --clock-control none): `{path}`", "",
             "Cold-cache, serialised per-launch times: compare shares, not absolutes.", "",
             "| kernel | launches | avg us | total us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / 1e3:.1f} | "
                     f"{sum(v) / tot * 100:.1f}% |")
    with open(dest, "w") as f:
        f.write("\n".join(lines) + "\n")
    print(dest)


def hbm(path, dest, peak_gbs=None):
    """Per-kernel achieved DRAM bandwidth from a launch list captured with
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum."""
    if peak_gbs is None:
        try:
            peak_gbs = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
        except (OSError, ValueError, KeyError):
            peak_gbs = 7700.0
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    ii = hdr.index("ID")
    per = defaultdict(dict)  # launch id -> metrics
    names = {}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
             "msecond": 1e6}
    for r in rows[1:]:
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
        per[r[ii]][r[mi]] = v
        names[r[ii]] = re.sub(r"\(.*", "", r[ki])[:70]
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for lid, m in per.items():
        a = agg[names[lid]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    lines = [f"# DRAM bandwidth per kernel (ncu launch list, --clock-control none): `{path}`", "",
             f"Peak = {peak_gbs} GB/s (MEASURED_PEAKS.json hbm_gbs). Per-launch times are serialised "
             "under ncu; tiny launches are latency-bound, compare the large ones.", "",
             "| kernel | launches | avg us | avg DRAM MB | GB/s | of peak |", "|---|---|---|---|---|---|"]
    for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        gbs = b / t if t else 0.0  # bytes / ns = GB/s
        lines.append(f"| `{k}` | {n} | {t / n / 1e3:.2f} | {b / n / 1e6:.2f} | {gbs:.0f} | "
                     f"{gbs / peak_gbs * 100:.0f}% |")
    with open(dest, "w") as f:
        f.write("\n".join(lines) + "\n")
    print(dest)


def movers(rep, dest, peak_gbs=None):
    """One row per launch of a --set full capture: duration, DRAM bytes, achieved GB/s, issue
    activity and the top warp-stall reasons (smsp__average_warps_issue_stalled_*)."""
    if peak_gbs is None:
        try:
            peak_gbs = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
        except (OSError, ValueError, KeyError):
            peak_gbs = 7700.0
    rows = ncu_csv(["-i", rep, "--page", "raw", "--csv"])
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1,
             "msecond": 1e3}

    def val(vals, key):
        if key not in hdr:
            return 0.0
        i = hdr.index(key)
        try:
            return float(vals[i].replace(",", "")) * scale.get(units[i], 1)
        except ValueError:
            return 0.0
    stall = [k for k in hdr if k.startswith("smsp__average_warps_issue_stalled_")
             and k.endswith("_per_issue_active.ratio") and "not_issued" not in k]
    lines = [f"# ncu --set full, one row per launch: `{rep}`", "",
             f"DRAM GB/s = (dram__bytes_read + dram__bytes_write) / gpu__time_duration; peak {peak_gbs} "
             "GB/s (MEASURED_PEAKS.json). Cold caches (ncu --cache-control all), serialised.", "",
             "| # | kernel | grid | us | DRAM MB | GB/s | of peak | issue active % | top stalls (warps per issue) |",
             "|---|---|---|---|---|---|---|---|---|"]
    for n, vals in enumerate(rows[2:]):
        name = re.sub(r"\(.*", "", vals[hdr.index("Kernel Name")]).replace("fusp::<unnamed>::", "")[:40]
        us = val(vals, "gpu__time_duration.sum")
        mb = (val(vals, "dram__bytes_read.sum") + val(vals, "dram__bytes_write.sum")) / 1e6
        gbs = mb * 1e6 / (us * 1e3) if us else 0.0
        issue = val(vals, "sm__inst_issued.avg.pct_of_peak_sustained_active")
        st = sorted(((val(vals, k), k) for k in stall), reverse=True)[:3]
        sts = ", ".join(f"{k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]} {v:.1f}"
                        for v, k in st if v > 0)
        grid = vals[hdr.index("launch__grid_size")] if "launch__grid_size" in hdr else ""
        lines.append(f"| {n} | `{name}` | {grid} | {us:.2f} | {mb:.2f} | {gbs:.0f} | "
                     f"{gbs / peak_gbs * 100:.0f}% | {issue:.1f} | {sts} |")
    with open(dest, "w") as f:
        f.write("\n".join(lines) + "\n")
    print(dest)


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    {"full": full, "launches": launches, "hbm": hbm, "movers": movers}[mode](src, dst)
