#!/usr/bin/env python
"""Run one workload point for a few windows (profiling helper).

  python tools/run_point.py c5_b32_T4.0_W4.0 --windows 1
  python tools/run_point.py c3 --windows 2
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402
from paper_cs_0405053_b200 import FLAG_DIGEST, IsingSR  # noqa: E402


def point(name):
    if name in workloads.CONFIGS:
        return workloads.get(name)
    for p in workloads.c5_points():
        if p.name == name:
            return p
    raise SystemExit(f"unknown point {name}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--windows", type=int, default=1)
    ap.add_argument("--skip", type=int, default=0)
    ap.add_argument("--profile", action="store_true", help="cudaProfilerStart after the skipped windows")
    args = ap.parse_args()
    w = point(args.name)
    sim = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), None if w.init == "random" else w.spins(), w.W, w.t_end,
                  w.seed, flags=FLAG_DIGEST)
    for k in range(args.skip + args.windows):
        if args.profile and k == args.skip:
            import torch
            torch.cuda.synchronize()
            torch.cuda.cudart().cudaProfilerStart()
        g = sim.run_window()
        ev = sim.commit()
        st = sim.stats()
        print(f"window {k}: g {g} events {ev} ms {st['ms_last_window']:.2f}", flush=True)
    sim.close()


if __name__ == "__main__":
    main()
