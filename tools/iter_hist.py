#!/usr/bin/env python
"""K1 time by worklist size over whole runs (where do big-region runs spend time?).

  python tools/iter_hist.py --config c3 [--b 32 --T 4 --W 4]   (c5 point: --config c5)
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads  # noqa: E402
from paper_cs_0405053_b200 import FLAG_LOG_EVENTS, IsingSR  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--b", type=int, default=32)
    ap.add_argument("--T", type=float, default=4.0)
    ap.add_argument("--W", type=float, default=4.0)
    ap.add_argument("--max-windows", type=int, default=1000)
    args = ap.parse_args()
    if args.config == "c5":
        w = [p for p in workloads.c5_points() if p.bx == args.b and p.T == args.T and p.W == args.W][0]
    else:
        w = workloads.get(args.config)
    torch.cuda.set_device(0)
    sim = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.spins(), w.W, w.t_end, w.seed, flags=FLAG_LOG_EVENTS)
    edges = [0, 64, 256, 1024, 4096, 16384, 1 << 30]
    ms = [0.0] * (len(edges) - 1)
    cnt = [0] * (len(edges) - 1)
    tot_events = 0
    nwin = 0
    while sim.stats()["t_c"] < w.t_end and nwin < args.max_windows:
        sim.begin_window()
        it = 0
        while True:
            it += 1
            s0 = sim.stats()
            ch, ov = sim.iterate()
            sim.exchange_done()
            s1 = sim.stats()
            n = s1["recomputations_total"] - s0["recomputations_total"]
            t = s1["region_ms"] - s0["region_ms"]
            for i in range(len(edges) - 1):
                if edges[i] <= n < edges[i + 1]:
                    ms[i] += t
                    cnt[i] += 1
            if ov:
                raise SystemExit("overflow")
            if not ch:
                sim.end_iterations(it)
                break
        tot_events += sim.commit()
        nwin += 1
    print(json.dumps({"workload": w.name, "windows": nwin, "events": tot_events,
                      "buckets": [{"regions": f"[{edges[i]},{edges[i + 1]})", "iterations": cnt[i],
                                   "k1_ms": round(ms[i], 2)} for i in range(len(ms))]}))


if __name__ == "__main__":
    main()
