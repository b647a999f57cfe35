#!/usr/bin/env python
"""Run a few windows of a warp-form workload (for ncu): c5 b32 T=4 W=1 on 8192^2,
windows `--skip` (untimed) then `--windows` inside cudaProfilerStart/Stop."""
import argparse, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import workloads  # noqa: E402
from paper_cs_0405053_b200 import FLAG_DIGEST, IsingSR  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--name", default="c5_b32_T4.0_W1.0")
ap.add_argument("--skip", type=int, default=2)
ap.add_argument("--windows", type=int, default=1)
args = ap.parse_args()
w = [p for p in workloads.c5_points() if p.name == args.name][0] if args.name.startswith("c5") else workloads.get(args.name)
torch.cuda.set_device(0)
sim = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.spins(), w.W, w.t_end, w.seed, flags=FLAG_DIGEST)
for _ in range(args.skip):
    sim.run_window(); sim.commit()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(args.windows):
    sim.run_window(); sim.commit()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(sim.stats()["g_last"])
