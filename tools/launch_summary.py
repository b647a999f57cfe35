#!/usr/bin/env python
"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per
kernel launches, total/mean device time and share of all kernel time."""
import csv
import collections
import sys


def main(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.reader(lines)
    hdr = next(rd)
    h = {k: i for i, k in enumerate(hdr)}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rd:
        if r[h["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[h["Kernel Name"]].split("(")[0]
        unit = r[h["Metric Unit"]]
        v = float(r[h["Metric Value"]].replace(",", ""))
        scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
        v_ms = v * scale.get(unit, 1.0)
        agg[name][0] += 1
        agg[name][1] += v_ms
    tot = sum(v[1] for v in agg.values())
    print(f"| kernel | launches | total ms | mean us | share |")
    print("|---|---|---|---|---|")
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {k} | {n} | {ms:.2f} | {1e3 * ms / n:.1f} | {ms / tot * 100:.1f}% |")
    print(f"\ntotal kernel time {tot:.2f} ms over {sum(v[0] for v in agg.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1])
