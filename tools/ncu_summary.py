#!/usr/bin/env python
"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel: count, total,
average, share.  Usage: python tools/ncu_summary.py launches.csv [--grid]"""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    gi = h.index("Grid Size") if "Grid Size" in h else None
    out = []
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1.0)
        name = r[ki].split("(")[0].replace("void ", "")
        out.append((name, v * scale, r[gi] if gi is not None else ""))
    return out


def main():
    data = load(sys.argv[1])
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, us, _ in data:
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':60s} {'launches':>8s} {'total_us':>11s} {'avg_us':>8s} {'share':>6s}")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:60]:60s} {n:8d} {t:11.1f} {t / n:8.2f} {t / tot:6.3f}")
    print(f"{'TOTAL':60s} {sum(v[0] for v in agg.values()):8d} {tot:11.1f}")


if __name__ == "__main__":
    main()
