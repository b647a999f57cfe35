#!/usr/bin/env python
"""Summarise an ncu report: key metrics per launch (stdout, markdown)."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("GPU Speed Of Light Throughput", "Duration"),
    ("GPU Speed Of Light Throughput", "Memory Throughput"),
    ("GPU Speed Of Light Throughput", "DRAM Throughput"),
    ("GPU Speed Of Light Throughput", "Compute (SM) Throughput"),
    ("Launch Statistics", "Grid Size"),
    ("Launch Statistics", "Registers Per Thread"),
    ("Occupancy", "Theoretical Occupancy"),
    ("Occupancy", "Achieved Occupancy"),
    ("Compute Workload Analysis", "Issued Ipc Active"),
    ("Scheduler Statistics", "No Eligible"),
    ("Warp State Statistics", "Warp Cycles Per Issued Instruction"),
    ("Warp State Statistics", "Avg. Active Threads Per Warp"),
    ("Memory Workload Analysis", "L1/TEX Hit Rate"),
    ("Memory Workload Analysis", "L2 Hit Rate"),
    ("Source Counters", "Branch Efficiency"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = {k: i for i, k in enumerate(rows[0])}
    by = {}
    for r in rows[1:]:
        by.setdefault(r[h["ID"]], {})[(r[h["Section Name"]], r[h["Metric Name"]])] = (r[h["Metric Value"]], r[h["Metric Unit"]])
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,"
                          "smsp__thread_inst_executed_per_inst_executed.ratio,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,"
                          "smsp__average_warp_latency_issue_stalled_long_scoreboard,smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct,"
                          "smsp__warp_issue_stalled_wait_per_warp_active.pct,smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct,"
                          "smsp__warp_issue_stalled_no_instruction_per_warp_active.pct,smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct,"
                          "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct,smsp__warp_issue_stalled_barrier_per_warp_active.pct"],
                         capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    print("| metric | " + " | ".join(f"launch {k}" for k in sorted(by, key=int)) + " |")
    print("|---|" + "---|" * len(by))
    for key in KEYS:
        vals = [" ".join(by[k].get(key, ("-", ""))) for k in sorted(by, key=int)]
        print(f"| {key[1]} | " + " | ".join(vals) + " |")
    if len(rr) > 2:
        hdr, units = rr[0], rr[1]
        for j, name in enumerate(hdr):
            if "__" in name:
                vals = [rr[i][j] for i in range(2, len(rr))]
                print(f"| {name} ({units[j]}) | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
