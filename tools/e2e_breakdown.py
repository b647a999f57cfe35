#!/usr/bin/env python
"""Where the end-to-end time of a c4 job goes: init (H2D + pack), each of the
first windows, the steady windows, the D2H of the final spins.

  python tools/e2e_breakdown.py [--config c4] [--windows 20]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads  # noqa: E402
from paper_cs_0405053_b200 import FLAG_DIGEST, IsingSR  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--windows", type=int, default=20)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    w = workloads.get(args.config)
    pinned = torch.from_numpy(w.spins()).pin_memory()
    pinned_out = torch.empty(w.Lx * w.Ly, dtype=torch.uint8).pin_memory()
    torch.cuda.synchronize()
    rec = {"config": args.config}
    t0 = time.perf_counter()
    sim = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), pinned.numpy(), w.W, w.t_end, w.seed, flags=FLAG_DIGEST)
    torch.cuda.synchronize()
    rec["init_s"] = time.perf_counter() - t0
    wins = []
    for k in range(args.windows):
        t1 = time.perf_counter()
        g = sim.run_window()
        ev = sim.commit()
        torch.cuda.synchronize()
        wins.append({"w": k, "g": g, "events": ev, "ms": 1e3 * (time.perf_counter() - t1)})
    for rep in range(2):  # the first call also loads the unpack kernel
        t2 = time.perf_counter()
        out = sim.spins(out=pinned_out.numpy())
        rec[f"d2h_s_{rep}"] = time.perf_counter() - t2
    rec["d2h_bytes"] = int(out.nbytes)
    st = sim.stats()
    sim.close()
    rec["windows"] = wins
    rec["region_ms_total"] = st["region_ms"]
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
