#!/usr/bin/env python
"""Benchmark: committed spin-flip events/s of the synchronous-relaxation
n-fold way (arXiv cs/0405053) on BASELINE config 4 (16384^2, 4x4 regions,
T=2, H=0, iid spins, W=0.5, t=50), strips over N GPUs.

A "step" is one window of committed time: the full relaxation to the fixed
point and the commit with the compacted event log (every §8(a) row).  W
warm-up windows, then K timed windows, continuing the same trajectory (t_end
is extended past 50 only if W+K > 100).  N > 1: one strip per GPU, the
library's own NCCL exchange (torch.distributed only broadcasts the NCCL id
and reduces the timings).

roofline: HBM, SURVEY §8(d.3)'s algorithmic bytes.  Per region and window
B_alg = A (S + 3H) + S + L with S the committed state (spins b^2/8 + halo
4b/8 + t_s 8 + R 8 + n 4 bytes), H = 4 + 9 h, L = 14 e, where A =
recomputations, h = boundary-history entries and e = committed events per
region per window, all measured by the run (ising_sr_stats).  The dominant
kernel K1 moves the A (S + 3H) part; `achieved` = those bytes / K1's device
time (CUDA events on the library's stream around every K1 launch).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ising|reference]

Prints one JSON line (rank 0).  --impl reference times the CPU oracle (the
reference arm of this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads  # noqa: E402

METRIC = "committed spin-flip events/s"
UNIT = "events/s"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "of fallback (B200_PROFILING.md: 6.65 TB/s, MEASURED_PEAKS.json absent)"


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def state_bytes(bx: int, by: int) -> float:
    """S of SURVEY §8(d.3): spins b^2/8 + halo (2bx + 2by)/8 + t_s 8 + R 8 + n 4."""
    return bx * by / 8.0 + (2 * bx + 2 * by) / 8.0 + 8 + 8 + 4


class WindowLedger:
    """Per-window A, h, e, g, f from ising_sr_stats after each commit, and the
    §8(d.3) algorithmic bytes they imply."""

    def __init__(self, w, nreg):
        self.S = state_bytes(w.bx, w.by)
        self.nreg = nreg
        self.rows = []

    def add(self, st):
        A_tot = float(sum(st["active_last"]))
        h = float(max(st["edge_entries_last_window"], 0))
        e = float(st["events_last_window"])
        H = 4.0 + 9.0 * h / self.nreg
        k1 = A_tot * (self.S + 3.0 * H)
        commit = self.nreg * self.S + 14.0 * e
        self.rows.append({"A": A_tot / self.nreg, "h": h / self.nreg, "e": e / self.nreg, "g": st["g_last"],
                          "f": st["f_last"], "k1_bytes": k1, "bytes": k1 + commit, "events": e,
                          "ms": st["ms_last_window"]})

    def total(self, key):
        return sum(r[key] for r in self.rows)

    def mean(self, key):
        return float(np.mean([r[key] for r in self.rows])) if self.rows else 0.0


# --------------------------------------------------------------------------
# clocks sampled during the timed region (B200_PROFILING.md recipe)
# --------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 5 + i and r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# --------------------------------------------------------------------------
# reference arm / cpu baseline: the oracle as it stands, on a bounded sample
# --------------------------------------------------------------------------
def oracle_sample(seconds_hint: float = 15.0):
    """c4's dynamics (T=2, H=0, 4x4 regions, iid start, same seed) on a
    2048^2 sub-lattice for t in [0, t_s); returns (events, wall s, sample)."""
    import oracle
    w = workloads.get("c4")
    L = 2048
    t_s = 1.0
    spins = workloads.initial_spins(L, L, "random", seed=w.seed)
    t0 = time.perf_counter()
    r = oracle.des_run(L, L, 4, 4, w.rates(), w.seed, spins, t_s)
    dt = time.perf_counter() - t0
    return r["n_events"], dt, f"oracle O1 on a {L}x{L} lattice (c4 dynamics: 4x4 regions, T=2, H=0), t in [0,{t_s})"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    try:
        os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
    except Exception:
        pass
    w = workloads.get("c4")
    L, t_win = 1024, w.W
    spins = workloads.initial_spins(L, L, "random", seed=w.seed)
    evs, secs = [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        r = oracle.des_run(L, L, 4, 4, w.rates(), w.seed, spins, t_win)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            evs.append(r["n_events"])
            secs.append(dt)
    val = sum(evs) / sum(secs)
    sample = f"oracle O1, one window [0,{t_win}) of c4 dynamics on a {L}x{L} sub-lattice per step"
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(secs) / len(secs),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "c4 sample: 1024^2 sub-lattice, 4x4 regions, T=2, H=0, iid +-1 seed 1, one window W=0.5"},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------
# the B200 arm
# --------------------------------------------------------------------------
def golden_parity(config, sim, world, nwin, w, rank=0, device=0, path=None):
    """The run against tests/golden/full_size/<config>_t50.json (the oracle's
    result, tools/make_goldens.py): total events, final spins and per-region
    event counts, bit for bit (SHA-256).  Only when the run ends exactly at
    the golden's t_end.  N > 1: the strips' spins and counts are hashed in
    rank order on rank 0 (received one strip at a time); every rank takes the
    same decisions, so the sends and receives match."""
    import hashlib
    path = path or os.path.join(ROOT, "tests", "golden", "full_size", f"{config}_t{int(w.t_end)}.json")
    if not os.path.exists(path):
        return None
    g = json.load(open(path))
    if abs(nwin * w.W - g["t_end"]) > 1e-12:
        return {"checked": False, "why": f"run ends at t = {nwin * w.W}, golden at {g['t_end']}"}
    _, cnt = sim.digests()
    spins = np.ascontiguousarray(sim.spins())
    cnt = np.ascontiguousarray(cnt.astype("<u8"))
    events = sim.stats()["events_total"]
    hs, hc = hashlib.sha256(), hashlib.sha256()
    if world == 1:
        hs.update(spins.tobytes())
        hc.update(cnt.tobytes())
    else:
        import torch
        import torch.distributed as dist
        dev = torch.device(f"cuda:{device}") if torch.cuda.is_available() else torch.device("cpu")  # (cpu: the gloo test)
        ev = torch.tensor([events], dtype=torch.int64, device=dev)
        dist.all_reduce(ev)
        events = int(ev.item())
        mine = [torch.from_numpy(spins.reshape(-1)).to(dev), torch.from_numpy(cnt.view(np.uint8).reshape(-1)).to(dev)]
        if rank == 0:
            hs.update(spins.tobytes())
            hc.update(cnt.tobytes())
            for r in range(1, world):  # equal strips: the same sizes on every rank
                for buf, h in zip(mine, (hs, hc)):
                    tmp = torch.empty_like(buf)
                    dist.recv(tmp, src=r)
                    h.update(tmp.cpu().numpy().tobytes())
        else:
            for buf in mine:
                dist.send(buf, dst=0)
            return None
    ok = {"events": events == g["n_events"],
          "spins": hs.hexdigest() == g["sha256_spins"], "counts": hc.hexdigest() == g["sha256_count"]}
    return {"checked": True, "bit_exact": all(ok.values()), **ok, "golden": os.path.relpath(path, ROOT)}


def run_ising(args):
    import torch
    from paper_cs_0405053_b200 import FLAG_DIGEST, FLAG_LOG_EVENTS, IsingSR

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # stdout carries the one JSON line
    nccl_id = None
    if world > 1:
        import torch.distributed as dist
        from paper_cs_0405053_b200.dist import shared_nccl_id
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        nccl_id = shared_nccl_id(rank)  # the library's own communicator does C1/C2

    w = workloads.get(args.config)
    if args.window == "tmax":  # the paper's T_max = ln N / (lambda |dG_i|)
        w = w.replace(W=workloads.paper_tmax(w.n_regions, workloads.boundary_sites(w.bx, w.by), max(w.rates())))
    nwin = args.warmup + args.steps
    t_end = max(w.t_end, nwin * w.W)
    spins = w.spins()
    # the commit compacts the window's event log (K3) inside the timed region;
    # per-region digests (a verification device, R27) only with --digest
    flags = FLAG_LOG_EVENTS | (FLAG_DIGEST if args.digest else 0)
    if args.jacobi_all:
        from paper_cs_0405053_b200 import FLAG_JACOBI_ALL
        flags |= FLAG_JACOBI_ALL
    if args.halo_loopback:  # one strip through the strip exchange to itself (a one-rank communicator)
        if world != 1:
            raise SystemExit("--halo-loopback is a one-GPU measurement of the strip exchange")
        from paper_cs_0405053_b200 import FLAG_HALO_LOOPBACK, nccl_unique_id
        flags |= FLAG_HALO_LOOPBACK
        nccl_id = nccl_unique_id()
    # the library's stream: every kernel of the path runs on it, and the
    # timing events are recorded on it
    stream = torch.cuda.Stream(device=local)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    sim = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), spins, w.W, t_end, w.seed, J=w.J, H=w.H, T=w.T,
                  flags=flags, rank=rank, world=world, device=local, stream=stream.cuda_stream, nccl_id=nccl_id,
                  torch_alloc=args.torch_alloc)
    for _ in range(args.warmup):
        sim.run_window()
        sim.commit()
    st0 = sim.stats()
    launches0 = sim.launch_count()
    ledger = WindowLedger(w, sim.n_regions)
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    gs = []
    ev = 0
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            gs.append(sim.run_window())
            ev += sim.commit()
            ledger.add(sim.stats())  # a host copy of the stats struct (no device work)
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1)
    st1 = sim.stats()
    launches = sim.launch_count() - launches0
    # whole-job numbers: events and bytes summed, time max over ranks
    tot_ev, max_ms = ev, ms
    region_ms = st1["region_ms"] - st0["region_ms"]
    impl_bytes = st1["region_bytes"] - st0["region_bytes"]
    nlaunch = st1["region_launches"] - st0["region_launches"]
    k1_bytes, alg_bytes = ledger.total("k1_bytes"), ledger.total("bytes")
    # steady state: the second half of the timed windows (device time of each window, ev0 -> ev1)
    half = ledger.rows[len(ledger.rows) // 2:]
    steady = {"windows": f"{nwin - len(half)}..{nwin - 1}",
              "events_per_s": sum(r["events"] for r in half) / max(sum(r["ms"] for r in half) * 1e-3, 1e-12)}
    # parity of the run with the oracle's golden result when the run ends at the config's t_end
    parity = golden_parity(args.config, sim, world, nwin, w, rank, local)
    compact_ms = st1["ms_compact_total"] - st0["ms_compact_total"]
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([float(ev), k1_bytes, alg_bytes, impl_bytes], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t)
        m = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        tot_ev, max_ms = int(t[0].item()), float(m[0].item())
        k1_bytes, alg_bytes, impl_bytes = (float(x) for x in t[1:].tolist())
    sim.close()

    # e2e: the public API from host buffers -- init (H2D of the lattice from
    # pinned memory + device packing) + K windows + D2H of the final spins
    e2e = None
    if not args.no_e2e:
        pinned = torch.from_numpy(spins).pin_memory()
        pinned_out = torch.empty((w.Ly // world) * w.Lx, dtype=torch.uint8).pin_memory()
        barrier()
        t0 = time.perf_counter()
        nccl_id2 = None
        if world > 1:  # a fresh ncclUniqueId for the second communicator
            from paper_cs_0405053_b200.dist import shared_nccl_id
            nccl_id2 = shared_nccl_id(rank)
        sim2 = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), pinned.numpy(), w.W, t_end, w.seed, flags=flags,
                       rank=rank, world=world, device=local, stream=stream.cuda_stream, nccl_id=nccl_id2,
                       torch_alloc=args.torch_alloc)
        ev2 = 0
        for _ in range(args.steps):
            sim2.run_window()
            ev2 += sim2.commit()
        out = sim2.spins(out=pinned_out.numpy())
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        sim2.close()
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([float(ev2), dt], dtype=torch.float64, device=f"cuda:{local}")
            dist.all_reduce(t[:1])
            dist.all_reduce(t[1:], op=dist.ReduceOp.MAX)
            ev2, dt = t[0].item(), t[1].item()
        e2e = {"value": ev2 / dt, "unit": UNIT,
               "h2d_bytes_per_step": spins.nbytes / args.steps,
               "d2h_bytes_per_step": (out.nbytes * world + 8 * args.steps) / args.steps,
               "includes": "ising_sr_init from pinned host spins (H2D + pack) + K windows + D2H of final spins",
               "device_buffers": ("torch caching allocator (blocks of the first context reused)" if args.torch_alloc
                                  else "cudaMalloc inside the timed region")}

    if rank != 0:
        return 0
    peak, peak_kind = _peaks()
    k1_alg_per_launch = k1_bytes / max(nlaunch, 1) / world
    achieved = (k1_bytes / world / (region_ms * 1e-3)) / 1e9 if region_ms > 0 else 0.0
    # DRAM bytes per K1 launch: the DRAM / §8(d.3)-algorithmic ratio of the
    # committed ncu capture of every K1 launch of one c4 window
    # (tools/ncu_traffic.py) times this run's algorithmic bytes per launch
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "k1_traffic_r08.json")
    if args.config == "c4" and os.path.exists(tp):
        t = json.load(open(tp))
        traffic = t["dram_over_alg"] * k1_alg_per_launch
        traffic_src = (f"profiles/k1_traffic_r08.json: ncu --set full of all {t['launches']} K1 launches of c4 "
                       f"window {t['window']}, DRAM / §8(d.3) K1 bytes = {t['dram_over_alg']:.2f}")
    window_bw = alg_bytes / (max_ms * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src, "peak_kind": peak_kind,
            "kernel": "K1 region_kernel<4,4> (+ region_kernel_first for each window's iteration 1)",
            "byte_model": "SURVEY §8(d.3): K1 moves A (S + 3H) per region per window; S, H, A, h measured",
            "bytes_per_launch": k1_alg_per_launch,
            "ms_per_launch": region_ms / max(nlaunch, 1),
            "share_of_step": region_ms / max_ms if max_ms > 0 else None,
            "window": {"bytes_alg_per_event": alg_bytes / max(tot_ev, 1), "achieved_gbs": window_bw,
                       "frac": window_bw / peak / world, "frac_vs_nominal_8000": window_bw / 8000.0 / world,
                       "formula": "B_alg = [A (S + 3H) + S + L] / e per committed event (SURVEY §8(d.3))"},
            "impl_bytes_per_event": impl_bytes / max(tot_ev, 1),
            "impl_bytes_note": "the library's own count of what K1 touches (DESIGN.md §6), not the roofline numerator"}
    # what actually bounds K1: instruction issue, not HBM -- the issue rate and lane
    # utilisation of the same committed ncu capture, as context beside the HBM fraction the metric asks for
    ip = os.path.join(ROOT, "profiles", "k1_issue_r08.json")
    if args.config == "c4" and os.path.exists(ip):
        t = json.load(open(ip))
        roof["issue"] = {"issued_ipc_active": t["issued_ipc_active_time_weighted"], "peak_ipc": t["peak_ipc"],
                         "frac": t["issued_ipc_active_time_weighted"] / t["peak_ipc"],
                         "active_lanes_per_warp_instruction": t["active_lanes_per_warp_instruction"],
                         "source": t["source"], "note": "from a capture under ncu, not measured in this run"}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        n_ev, secs, sample = oracle_sample()
        cpu = {"value": n_ev / secs, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
               "cpu_model": _cpu_model(), "host_cores": os.cpu_count()}
    line = {
        "metric": METRIC, "value": tot_ev / (max_ms * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": max_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{args.config}: {w.Lx}x{w.Ly} periodic, {w.bx}x{w.by} regions, T={w.T}, H={w.H}, "
                               f"iid +-1 seed {w.seed}, W={w.W}, windows {args.warmup}..{nwin - 1} "
                               f"(t {args.warmup * w.W}..{nwin * w.W})",
                   "regions": w.n_regions, "l2": "inputs larger than L2 (state+histories >> 126 MB)",
                   "schedule": "jacobi_all" if args.jacobi_all else "worklist",
                   "event_log": "compacted at every commit (FLAG_LOG_EVENTS), in the timed region",
                   "digests": bool(args.digest),
                   "parallelism": f"strips{world}",
                   "exchange": (None if world == 1 and not args.halo_loopback else
                                os.environ.get("ISING_SR_EXCHANGE", "peer") + (" (loopback)" if args.halo_loopback else ""))},
        "events": tot_ev,
        "iterations_per_window": {"mean": float(np.mean(gs)), "p50": float(np.percentile(gs, 50)),
                                  "p99": float(np.percentile(gs, 99)), "max": int(max(gs)), "min": int(min(gs)),
                                  "ln_N": math.log(w.n_regions),
                                  "paper_tmax": workloads.paper_tmax(w.n_regions, workloads.boundary_sites(w.bx, w.by),
                                                                     max(w.rates()))},
        "per_region_per_window": {"A_recomputations": ledger.mean("A"), "h_edge_entries": ledger.mean("h"),
                                  "e_events": ledger.mean("e"), "S_state_bytes": ledger.S,
                                  "f_max": int(max(r["f"] for r in ledger.rows))},
        "commit_compaction_ms_per_window": compact_ms / args.steps,
        "steady_state_second_half": steady,
        "parity": parity,
        "gpu_launches": launches,
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


# --------------------------------------------------------------------------
# second workload (--config cb): checkerboard Metropolis sweeps of the c4
# lattice (16384^2, T = 2, H = 0, seed 1); a step = one sweep (both colours)
# --------------------------------------------------------------------------
CB_OPS_PER_SITE = 45  # integer ops of one visit: half a Philox4x32-10 draw (10 rounds x 7 / 2) + U, class, compare


def run_cb(args):
    import torch
    from paper_cs_0405053_b200 import checkerboard_run, checkerboard_sweeps

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1 and rank != 0:
        return 0  # replicas only: one lattice per GPU needs no exchange we measure here
    torch.cuda.set_device(0)
    w = workloads.get("c4")
    Lx, Ly, p, seed = w.Lx, w.Ly, w.rates(), w.seed
    n = Lx * Ly
    spins = w.spins()
    stream = torch.cuda.current_stream()
    d = torch.from_numpy(spins.reshape(-1).copy()).cuda()
    fl = torch.zeros(1, dtype=torch.int64, device="cuda")
    checkerboard_sweeps(d.data_ptr(), Lx, Ly, p, seed, 0, args.warmup, fl.data_ptr(), stream.cuda_stream)
    torch.cuda.synchronize()
    f0 = int(fl.item())
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        e0.record(stream)
        checkerboard_sweeps(d.data_ptr(), Lx, Ly, p, seed, args.warmup, args.steps, fl.data_ptr(),
                            stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    flips = int(fl.item()) - f0
    value = n * args.steps / (ms * 1e-3)
    e2e = None
    if not args.no_e2e:
        pin_in = torch.from_numpy(spins.reshape(-1).copy()).pin_memory()
        pin_out = torch.empty(n, dtype=torch.uint8).pin_memory()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, _ = checkerboard_run(pin_in.numpy(), Lx, Ly, p, seed, 0, args.steps, out=pin_out.numpy())
        dt = time.perf_counter() - t0
        e2e = {"value": n * args.steps / dt, "unit": "site updates/s", "h2d_bytes_per_step": n / args.steps,
               "d2h_bytes_per_step": (n + 8) / args.steps,
               "includes": "ising_cb_run from pinned host spins: device alloc + H2D + K sweeps + D2H"}
    clocks = clk.summary()
    f_mhz = clocks.get("sm_max_mhz") or 1965.0
    peak = 148 * 128 * f_mhz * 1e6 / 1e12  # Tops/s: 4 SMSPs x (fma + alu pipe) x 16 lanes per clock
    achieved = CB_OPS_PER_SITE * n * args.steps / (ms * 1e-3) / 1e12
    cpu = None
    if not args.no_cpu_baseline:
        import oracle
        sub = workloads.initial_spins(2048, 2048, "random", seed)
        t0 = time.perf_counter()
        oracle.cb_run(sub, 2048, 2048, p, seed, 0, 4)
        secs = time.perf_counter() - t0
        cpu = {"value": 2048 * 2048 * 4 / secs, "unit": "site updates/s", "cores": 1, "kind": "oracle",
               "sample": "orc_cb_run, 2048^2 sub-lattice of the same dynamics (T=2), 4 sweeps"}
    line = {
        "metric": "checkerboard Metropolis site updates/s", "value": value, "unit": "site updates/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8+f64",
        "data": "synthetic",
        "config": {"workload": f"cb: {Lx}x{Ly} periodic checkerboard Metropolis, T={w.T}, H={w.H}, iid +-1 seed {seed}, "
                               f"sweeps {args.warmup}..{args.warmup + args.steps - 1}",
                   "l2": "lattice (268 MB) larger than L2", "parallelism": "single GPU"},
        "flips": flips, "acceptance": flips / (n * args.steps),
        "gpu_launches": 2 * args.steps,
        "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Tops/s",
                     "frac": achieved / peak, "traffic": None,
                     "ops_per_site": CB_OPS_PER_SITE,
                     "peak_kind": "derived: 148 SMs x 128 int lanes/clk (fma + alu pipes) x max SM clock",
                     "kernel": "half_sweep_w (both colours)"},
        "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=97)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ising", choices=["ising", "reference"])
    ap.add_argument("--config", default="c4")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--torch-alloc", action=argparse.BooleanOptionalAction, default=True,
                    help="device buffers from torch's caching allocator (binding option torch_alloc; the e2e context "
                         "then reuses the blocks the first context returned instead of fresh cudaMalloc calls, whose "
                         "cost varied 50-450 ms between boxes); --no-torch-alloc: the library's own cudaMalloc")
    ap.add_argument("--digest", action="store_true", help="also maintain the per-region event digests")
    ap.add_argument("--window", default="config", choices=["config", "tmax"],
                    help="W of the config, or the paper's T_max = ln N/(lambda |dG|) (P:502-515)")
    ap.add_argument("--halo-loopback", action="store_true",
                    help="N=1: run the strip exchange to itself (ISING_SR_EXCHANGE=peer|sendrecv picks the transport)")
    ap.add_argument("--jacobi-all", action="store_true",
                    help="paper-faithful schedule: every region in every iteration (same bits and g)")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.config == "cb":
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "the cb workload's reference arm is the oracle "
                              "timed in its cpu_baseline"}))
            return 0
        return run_cb(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ising(args)


if __name__ == "__main__":
    sys.exit(main())
