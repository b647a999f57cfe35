#!/usr/bin/env python
"""Per-iteration profile of a window: regions recomputed, events, kernel ms.

  python tools/iter_profile.py [--config c4] [--skip 3] [--windows 2]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads  # noqa: E402
from paper_cs_0405053_b200 import FLAG_DIGEST, FLAG_LOG_EVENTS, IsingSR  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--skip", type=int, default=3)
    ap.add_argument("--windows", type=int, default=2)
    ap.add_argument("--W", type=float, default=None)
    ap.add_argument("--profile", action="store_true", help="cudaProfilerStart before the measured windows")
    args = ap.parse_args()
    w = workloads.get(args.config)
    if args.W:
        w = w.replace(W=args.W)
    torch.cuda.set_device(0)
    sim = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.spins(), w.W, w.t_end, w.seed, flags=FLAG_DIGEST | FLAG_LOG_EVENTS)
    for _ in range(args.skip):
        sim.run_window()
        sim.commit()
    out = []
    if args.profile:
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
    for k in range(args.windows):
        sim.begin_window()
        rows = []
        it = 0
        while True:
            it += 1
            s0 = sim.stats()
            ch, ov = sim.iterate()
            sim.exchange_done()
            s1 = sim.stats()
            rows.append({"it": it, "regions": s1["recomputations_total"] - s0["recomputations_total"],
                         "ms": round(s1["region_ms"] - s0["region_ms"], 4),
                         "MB": round((s1["region_bytes"] - s0["region_bytes"]) / 1e6, 2)})
            if ov:
                raise SystemExit("overflow")
            if not ch:
                sim.end_iterations(it)
                break
        ev = sim.commit()
        st = sim.stats()
        S = w.bx * w.by / 8 + (2 * w.bx + 2 * w.by) / 8 + 20  # SURVEY §8(d.3) committed state bytes
        out.append({"window": args.skip + k, "events": ev, "iters": rows, "nreg": sim.n_regions,
                    "h": st["edge_entries_last_window"], "S": S})
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
