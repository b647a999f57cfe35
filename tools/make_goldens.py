"""Write full-size golden results of the CPU oracle to tests/golden/full_size/.

Calls only `oracle/` (the plain serial DES) and `workloads/`
(the seeded inputs): nothing here touches the CUDA library.  The trajectory
of the per-region-stream dynamics does not depend on the window W (the
windows only schedule the relaxation), so one oracle run per
(lattice, region size, T, H, t_end) covers every W of that point.

For every trajectory the file records the number of events, SHA-256 of the
final spins (row-major u8), of the per-region digests (u64 little-endian,
DESIGN.md R27) and of the per-region event counts (u64 LE), the first
regions' digests in hex (for diagnosis), and the oracle's wall time on one
host core.  tests/test_gpu_goldens.py compares the GPU against these.

    python tools/make_goldens.py [--jobs 6] [--only NAME ...] [--list]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import multiprocessing as mp
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tests", "golden", "full_size")


def trajectories():
    """(name, workload, t_end, cost estimate) for every golden trajectory."""
    import workloads
    out = []
    c3 = workloads.get("c3")
    out.append(("c3_t200", c3, 200.0, 3e7))
    c4 = workloads.get("c4")
    out.append(("c4_t1", c4, 1.0, 1.5e8))
    out.append(("c4_t50", c4, 50.0, 2.5e9))
    rho = {1.0: 0.19, 2.269: 0.35, 4.0: 0.63}
    for b in (1, 2, 4, 8, 32):
        for T in (1.0, 2.269, 4.0):
            w = workloads.Workload(f"c5_b{b}_T{T}", 8192, 8192, b, b, T=T, W=1.0, t_end=16.0)
            # the heap over 67M 1x1 regions costs several times more per event
            cost = rho[T] * 8192 * 8192 * 16 * (4.0 if b == 1 else 1.5 if b == 2 else 1.0)
            out.append((f"c5_b{b}_T{T}", w, 16.0, cost))
    return out


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.machine()


def sha(a) -> str:
    return hashlib.sha256(a.tobytes()).hexdigest()


def run_one(item):
    name, w, t_end, _ = item
    import numpy as np

    import oracle
    path = os.path.join(OUT, name + ".json")
    if os.path.exists(path):
        return name, "exists"
    spins0 = w.spins()
    t0 = time.time()
    ref = oracle.des_run(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.seed, spins0, t_end)
    wall = time.time() - t0
    dig = np.ascontiguousarray(ref["digest"], dtype="<u8")
    cnt = np.ascontiguousarray(ref["count"], dtype="<u8")
    rec = {
        "name": name,
        "workload": {"Lx": w.Lx, "Ly": w.Ly, "bx": w.bx, "by": w.by, "T": w.T, "J": w.J, "H": w.H,
                     "init": w.init, "seed": w.seed, "rule": w.rule},
        "t_end": t_end,
        "n_events": int(ref["n_events"]),
        "n_regions": int(dig.size),
        "sha256_spins": sha(np.ascontiguousarray(ref["spins"], dtype=np.uint8)),
        "sha256_digest": sha(dig),
        "sha256_count": sha(cnt),
        "digest_head": [f"{int(x):016x}" for x in dig[:8]],
        "count_head": [int(x) for x in cnt[:8]],
        "up_sites": int(np.count_nonzero(ref["spins"])),
        "oracle_wall_s": round(wall, 1),
        "oracle_events_per_s": round(ref["n_events"] / wall, 1) if wall > 0 else None,
        "host": _cpu_model(),
        "generator": "tools/make_goldens.py (oracle/ only)",
    }
    tmp = path + ".tmp"
    with open(tmp, "w") as f:
        json.dump(rec, f, indent=1)
    os.replace(tmp, path)
    return name, f"{rec['n_events']} events in {wall:.0f} s"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=6)
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--list", action="store_true")
    args = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    items = trajectories()
    if args.only:
        items = [t for t in items if t[0] in args.only]
    if args.list:
        for t in items:
            print(t[0], t[2], f"{t[3]:.2e}")
        return
    import oracle
    oracle.build()
    items.sort(key=lambda t: -t[3])  # longest first
    with mp.get_context("fork").Pool(args.jobs) as pool:
        for name, msg in pool.imap_unordered(run_one, items):
            print(f"{time.strftime('%H:%M:%S')} {name}: {msg}", flush=True)


if __name__ == "__main__":
    main()
