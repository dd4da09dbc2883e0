#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: time per kernel family."""
import csv
import re
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.DictReader(l for l in open(path) if not l.startswith("==")))
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        key = re.sub(r"\(.*", "", name)
        m = re.match(r"void pqb::k_gemm<(.*?)>", name)
        if m:
            key = "k_gemm<" + m.group(1) + ">"
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        us = {"ns": v / 1e3, "nsecond": v / 1e3, "us": v, "usecond": v, "ms": v * 1e3, "msecond": v * 1e3}[unit]
        agg[key][0] += 1
        agg[key][1] += us
        total += us
    print(f"{'kernel':70s} {'launches':>8s} {'total_us':>10s} {'share':>6s}")
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:70]:70s} {n:8d} {us:10.1f} {100 * us / total:5.1f}%")
    print(f"{'TOTAL':70s} {sum(v[0] for v in agg.values()):8d} {total:10.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
