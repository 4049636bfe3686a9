#!/usr/bin/env python
"""Summarise ncu CSV output for profiles/.

    python tools/ncu_summary.py launches <launches.csv>        # per-kernel share table
    python tools/ncu_summary.py raw <raw.csv> [bytes_per_launch] # --page raw metrics of a capture
"""

from __future__ import annotations

import collections
import csv
import io
import re
import sys


def _rows(path):
    text = open(path, errors="replace").read()
    start = text.find('"ID"')
    return list(csv.DictReader(io.StringIO(text[start:])))


def short(name):
    name = re.sub(r"\(bool\)", "", name)
    name = name.replace("void ", "")
    m = re.match(r"([\w:]+(<[^()]*>)?)", name)
    base = m.group(1) if m else name
    if "at::" in base or "at::native" in name:
        return "torch: " + base.split("<")[0][:60]
    return base


def launches(path):
    rows = [r for r in _rows(path) if r.get("Metric Name") == "gpu__time_duration.sum"]
    agg = collections.OrderedDict()
    total = 0.0
    for r in rows:
        k = short(r["Kernel Name"])
        t = float(r["Metric Value"].replace(",", ""))
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += t
        total += t
    print(f"{len(rows)} launches, {total / 1e6:.3f} ms total (cold-cache, serialised)\n")
    print("| kernel | launches | total ms | mean us | share |")
    print("|---|---:|---:|---:|---:|")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {c} | {t / 1e6:.3f} | {t / c / 1e3:.1f} | {100 * t / total:.1f}% |")


def raw(path, algo_bytes=None):
    rows = _rows(path)
    keys = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "lts__t_sector_hit_rate.pct",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__t_sector_hit_rate.pct", "launch__occupancy_limit_registers"]
    for r in rows[1:] if rows and rows[0].get("ID") == "" else rows:
        name = short(r.get("Kernel Name", "?"))
        vals = {k: r.get(k) for k in keys if k in r}
        print(name, vals)
        try:
            rd = float(vals["dram__bytes_read.sum"].replace(",", ""))
            wr = float(vals["dram__bytes_write.sum"].replace(",", ""))
            print(f"  traffic {rd + wr:.4g} B", end="")
            if algo_bytes:
                print(f"  ({(rd + wr) / float(algo_bytes):.3f} x algorithmic)", end="")
            print()
        except (KeyError, ValueError, AttributeError):
            pass


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        raw(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
