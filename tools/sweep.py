#!/usr/bin/env python
"""Per-config reports: committed events/s, iterations per window g (vs ln N),
f, recomputations per region per window, and (with --oracle) the oracle's
events/s and bit-exact parity on the same full run.

  python tools/sweep.py --configs c1,c2,c3 --oracle --out profiles/r01_configs.jsonl
  python tools/sweep.py --c5 [--only b32] --out profiles/r01_c5_sweep.jsonl [--csv profiles/r01_c5_sweep.csv]
  python tools/sweep.py --c5 --golden ...   # parity against tests/golden/full_size (oracle goldens)
  python tools/sweep.py --c5 --window tmax  # the paper's W = T_max = ln N / (lambda |dG|) per point

Device time = CUDA events around the run_window + commit calls (inputs
resident); g, f and recomputations come from ising_sr_stats.
"""
import argparse
import csv
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_cs_0405053_b200 import FLAG_DIGEST, IsingSR  # noqa: E402


MAX_IT = 0  # 0: the library's default (1000)


def run_one(w, digest=True):
    stream = torch.cuda.Stream()
    sim = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.spins(), w.W, w.t_end, w.seed, J=w.J, H=w.H, T=w.T,
                  flags=FLAG_DIGEST if digest else 0, stream=stream.cuda_stream, max_iterations=MAX_IT)
    gs, fs, evs, wms = [], [], [], []
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(w.n_windows()):
        gs.append(sim.run_window())
        evs.append(sim.commit())
        st = sim.stats()
        fs.append(st["f_last"])
        wms.append(st["ms_last_window"])
    e1.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ms = e0.elapsed_time(e1)
    st = sim.stats()
    out = {"sim": sim, "g": gs, "f": fs, "events": evs, "ms": ms, "wall_s": wall, "stats": st, "window_ms": wms}
    return out


def record(w, r):
    g = np.array(r["g"])
    N = w.n_regions
    bd = 1 if (w.bx == 1 and w.by == 1) else 2 * (w.bx + w.by) - 4
    tot = int(sum(r["events"]))
    st = r["stats"]
    return {
        "config": w.name, "Lx": w.Lx, "Ly": w.Ly, "bx": w.bx, "by": w.by, "T": w.T, "H": w.H, "W": w.W,
        "t_end": w.t_end, "regions": N, "ln_N": math.log(N), "windows": len(g),
        "events": tot, "device_s": r["ms"] / 1e3, "events_per_s": tot / (r["ms"] / 1e3),
        "wall_events_per_s": tot / r["wall_s"],
        "g_mean": float(g.mean()), "g_p50": float(np.percentile(g, 50)), "g_p99": float(np.percentile(g, 99)),
        "g_max": int(g.max()), "f_mean": float(np.mean(r["f"])), "f_max": int(max(r["f"])),
        "recomputations_per_region_window": st["recomputations_total"] / (N * len(g)),
        "events_per_region_window": tot / (N * len(g)),
        "paper_T_max": math.log(N) / bd,  # T_max = ln N / (lambda |dG|), lambda = 1
        "hist_capacity": st["hist_capacity"], "overflow_retries": st["overflow_retries"],
        "gpu": torch.cuda.get_device_name(0),
        "window_ms": [round(x, 3) for x in r["window_ms"]], "window_events": [int(x) for x in r["events"]],
        "window_g": [int(x) for x in r["g"]],
    }


def golden_name(w):
    if w.name.startswith("c5_"):
        return "_".join(w.name.split("_")[:3])  # c5_b{b}_T{T}: one trajectory for every W
    return {"c3": "c3_t200", "c4": "c4_t50"}.get(w.name)


def golden_parity(w, sim, total):
    """Bit-exact check against tests/golden/full_size/<trajectory>.json (the
    oracle's SHA-256 of final spins, per-region digests and counts)."""
    import hashlib
    name = golden_name(w)
    path = os.path.join(ROOT, "tests", "golden", "full_size", f"{name}.json")
    if not name or not os.path.exists(path):
        return None
    g = json.load(open(path))
    if g["t_end"] != w.t_end:
        return None
    dig, cnt = sim.digests()
    sh = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    return bool(total == g["n_events"] and sh(cnt.astype("<u8")) == g["sha256_count"]
                and sh(dig.astype("<u8")) == g["sha256_digest"] and sh(sim.spins()) == g["sha256_spins"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="")
    ap.add_argument("--c5", action="store_true")
    ap.add_argument("--only", default="")
    ap.add_argument("--oracle", action="store_true", help="also run the CPU oracle (test infrastructure) for parity")
    ap.add_argument("--golden", action="store_true", help="bit-exact parity against tests/golden/full_size")
    ap.add_argument("--window", default="config", choices=["config", "tmax"])
    ap.add_argument("--max-iterations", type=int, default=0)
    ap.add_argument("--out", required=True)
    ap.add_argument("--csv", default="")
    args = ap.parse_args()
    global MAX_IT
    MAX_IT = args.max_iterations
    torch.cuda.set_device(0)
    ws = [workloads.get(c) for c in args.configs.split(",") if c]
    if args.c5:
        ws += [p for p in workloads.c5_points() if args.only in p.name]
    if args.window == "tmax":  # the paper's window, one run per (b, T)
        seen, tw = set(), []
        for w in ws:
            key = (w.bx, w.by, w.T, w.name.split("_W")[0])
            if key in seen:
                continue
            seen.add(key)
            W = workloads.paper_tmax(w.n_regions, workloads.boundary_sites(w.bx, w.by), max(w.rates()))
            tw.append(w.replace(W=W, name=f"{key[3]}_Wtmax"))
        ws = tw
    rows = []
    with open(args.out, "a") as fo:
        for w in ws:
            try:
                r = run_one(w)
            except Exception as e:  # e.g. E_OOM for a point that does not fit: record it, go on
                rec = {"config": w.name, "W": w.W, "error": str(e)}
                rows.append(rec)
                fo.write(json.dumps(rec) + "\n")
                fo.flush()
                print(json.dumps(rec), flush=True)
                torch.cuda.empty_cache()
                continue
            rec = record(w, r)
            if args.golden:
                rec["parity_golden"] = golden_parity(w, r["sim"], rec["events"])
            if args.oracle:
                import oracle
                dig, cnt = r["sim"].digests()
                spins = r["sim"].spins()
                t0 = time.perf_counter()
                ref = oracle.des_workload(w)
                dt = time.perf_counter() - t0
                rec["oracle_events_per_s"] = ref["n_events"] / dt
                rec["oracle_cores"] = 1
                rec["parity_bit_exact"] = bool(ref["n_events"] == rec["events"] and np.array_equal(cnt, ref["count"])
                                               and np.array_equal(spins, ref["spins"])
                                               and np.array_equal(dig, ref["digest"]))
            r["sim"].close()
            rows.append(rec)
            fo.write(json.dumps(rec) + "\n")
            fo.flush()
            print(json.dumps(rec), flush=True)
    if args.csv:
        keys = list(rows[0].keys())
        with open(args.csv, "w", newline="") as f:
            wr = csv.DictWriter(f, fieldnames=keys, extrasaction="ignore")
            wr.writeheader()
            for r in rows:
                wr.writerow(r)


if __name__ == "__main__":
    main()
