#!/usr/bin/env python
"""Markdown table of selected ncu --page details metrics (one column per
profiled launch) from `ncu -i REP --page details --csv > DETAILS.csv`.

  python tools/ncu_details_md.py DETAILS.csv TITLE [--labels a,b,...] >> OUT.md
"""
import csv
import sys

METRICS = ["Duration", "Grid Size", "Block Size", "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy",
           "Issued Ipc Active", "No Eligible", "Avg. Active Threads Per Warp", "Branch Efficiency",
           "Executed Instructions", "DRAM Throughput", "Compute (SM) Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
           "Warp Cycles Per Issued Instruction"]


def main():
    path, title = sys.argv[1], sys.argv[2]
    labels = sys.argv[sys.argv.index("--labels") + 1].split(",") if "--labels" in sys.argv else None
    rows = list(csv.reader(open(path)))
    h = rows[0]
    iid, iname, imet, ival, iunit = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    by = {}
    names = {}
    for r in rows[1:]:
        if len(r) <= ival:
            continue
        by.setdefault(r[iid], {})[r[imet]] = (r[ival] + " " + r[iunit]).strip()
        names[r[iid]] = r[iname]
    ids = sorted(by, key=int)
    labels = labels or [f"launch {i}" for i in ids]
    print(f"## {title}\n")
    print("kernels: " + "; ".join(sorted(set(n.split("(")[0] for n in names.values()))) + "\n")
    print("| metric | " + " | ".join(labels) + " |")
    print("|---|" + "---|" * len(ids))
    for m in METRICS:
        print(f"| {m} | " + " | ".join(by[i].get(m, "") for i in ids) + " |")
    print()


if __name__ == "__main__":
    main()
