#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
launches, total and mean time and share per kernel.

  python tools/launch_summary.py LAUNCHES.csv [--md OUT.md]
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    md = sys.argv[sys.argv.index("--md") + 1] if "--md" in sys.argv else None
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    ik, iv, iu, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Metric Name")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        name = r[ik].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | total ms | mean us | share |", "|---|---|---|---|---|"]
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| {k} | {n} | {ms:.2f} | {1e3 * ms / n:.1f} | {100 * ms / tot:.1f}% |")
    out.append(f"\ntotal kernel time {tot:.2f} ms over {sum(v[0] for v in agg.values())} launches")
    txt = "\n".join(out)
    print(txt)
    if md:
        open(md, "w").write(txt + "\n")


if __name__ == "__main__":
    main()
