#!/usr/bin/env python
"""Where a whole run's time goes: per-window device time (ms_last_window) against
K1 (region_ms), the commit's log compaction (ms_compact_total) and the
regions replayed at commit, for one config (default c3), with the event log.

  python tools/time_split.py [--config c3] [--no-log]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads  # noqa: E402
from paper_cs_0405053_b200 import FLAG_LOG_EVENTS, IsingSR, IsingSRError  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--no-log", action="store_true")
    args = ap.parse_args()
    w = workloads.get(args.config)
    torch.cuda.set_device(0)
    sim = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.spins(), w.W, w.t_end, w.seed,
                  flags=0 if args.no_log else FLAG_LOG_EVENTS)
    tot = {"window_ms": 0.0, "k1_ms": 0.0, "compact_ms": 0.0, "replayed": 0, "iterations": 0, "windows": 0, "events": 0}
    early = None
    while True:
        try:
            sim.run_window()
        except IsingSRError as e:
            if e.status == -9:
                break
            raise
        s0 = sim.stats()
        tot["events"] += sim.commit()
        s = sim.stats()
        tot["windows"] += 1
        tot["window_ms"] += s["ms_last_window"]
        tot["replayed"] += max(0, s["log_replayed_last_window"])
        if tot["windows"] == 5:
            early = dict(tot, k1_ms=s["region_ms"], compact_ms=s["ms_compact_total"], iterations=s["iterations_total"])
    s = sim.stats()
    tot.update(k1_ms=s["region_ms"], compact_ms=s["ms_compact_total"], iterations=s["iterations_total"])
    print(json.dumps({"config": args.config, "log": not args.no_log, "total": tot, "first5": early}))


if __name__ == "__main__":
    main()
