#!/usr/bin/env python
"""Iterations per window g against ln N (the paper's Theorem 2).

Fixed region size b x b and temperature, lattices L = 2^k so N = (L/b)^2
regions; for each N two windows: the paper's T_max = ln N / (lambda |dG|)
(lambda = 1, |dG| = 4b - 4) and a fixed W.  Records g (mean, p50,
max over the windows after a warm-up of `--skip` windows), A and events/s.

  python tools/gscaling.py --out profiles/r01_g_vs_lnN.jsonl [--b 4] [--T 2.269]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_cs_0405053_b200 import IsingSR  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--b", type=int, default=4)
    ap.add_argument("--T", type=float, default=2.269)
    ap.add_argument("--W", type=float, default=0.5)
    ap.add_argument("--L", default="64,128,256,512,1024,2048,4096,8192,16384")
    ap.add_argument("--windows", type=int, default=8)
    ap.add_argument("--skip", type=int, default=4)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    b = args.b
    dG = 1 if b == 1 else 4 * b - 4
    with open(args.out, "a") as fo:
        for L in [int(x) for x in args.L.split(",")]:
            N = (L // b) ** 2
            for kind, W in (("T_max", math.log(N) / dG), ("fixed", args.W)):
                w = workloads.Workload(f"g_L{L}_{kind}", L, L, b, b, T=args.T, W=W,
                                       t_end=W * (args.skip + args.windows), seed=1)
                sim = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.spins(), w.W, w.t_end, w.seed)
                gs, evs = [], []
                st0 = None
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                for k in range(args.skip + args.windows):
                    if k == args.skip:
                        st0 = sim.stats()
                        e0.record()
                    g = sim.run_window()
                    ev = sim.commit()
                    if k >= args.skip:
                        gs.append(g)
                        evs.append(ev)
                e1.record()
                torch.cuda.synchronize()
                st1 = sim.stats()
                sim.close()
                g = np.array(gs)
                rec = {"L": L, "b": b, "T": args.T, "regions": N, "ln_N": math.log(N), "W_kind": kind, "W": W,
                       "paper_T_max": math.log(N) / dG, "g_mean": float(g.mean()), "g_p50": float(np.median(g)),
                       "g_max": int(g.max()),
                       "A": (st1["recomputations_total"] - st0["recomputations_total"]) / (N * args.windows),
                       "events_per_region_window": sum(evs) / (N * args.windows),
                       "events_per_s": sum(evs) / (e0.elapsed_time(e1) * 1e-3),
                       "windows": f"{args.skip}..{args.skip + args.windows - 1}"}
                fo.write(json.dumps(rec) + "\n")
                fo.flush()
                print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
