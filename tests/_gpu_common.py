"""Shared helpers of the GPU parity tests: run a workload through the C ABI
(binding.IsingSR) window by window, and compare it with the CPU oracle bit
for bit."""
import numpy as np

import oracle
from paper_cs_0405053_b200 import FLAG_DIGEST, FLAG_LOG_EVENTS, IsingSR, IsingSRError


def run_gpu(w, flags=FLAG_DIGEST | FLAG_LOG_EVENTS, per_window_logs=False, **kw):
    sim = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.spins(), w.W, w.t_end, w.seed, flags=flags, **kw)
    logs, gs, wstats = [], [], []
    total = 0
    while True:
        try:
            g = sim.run_window()
        except IsingSRError as e:
            if e.status == -9:  # past t_end
                break
            raise
        gs.append(g)
        total += sim.commit()
        if per_window_logs:
            logs.append(sim.events())
            wstats.append(sim.stats())
    dig, cnt = sim.digests()
    out = {"spins": sim.spins(), "digest": dig, "count": cnt, "events": total, "g": gs,
           "logs": logs, "stats": sim.stats(), "window_stats": wstats}
    sim.close()
    return out


def check_against_oracle(w, gpu=None, logs=True, oracle_kw=None, **gpu_kw):
    """The GPU run of workload w (or `gpu`) against the oracle: total events,
    per-region counts and digests, final spins, and (logs) every window's
    compact event log entry by entry."""
    ref = oracle.des_workload(w, log_cap=10**7 if logs else 0, **(oracle_kw or {}))
    gpu = gpu or run_gpu(w, per_window_logs=logs, **gpu_kw)
    assert gpu["events"] == ref["n_events"]
    assert np.array_equal(gpu["count"], ref["count"])
    assert np.array_equal(gpu["spins"], ref["spins"])
    if gpu["digest"] is not None:
        assert np.array_equal(gpu["digest"], ref["digest"])
    if logs and gpu["logs"]:
        # window w holds the oracle events with t in [fl(w W), fl((w+1) W))
        t_all, r_all, s_all = ref["log_t"], ref["log_region"], ref["log_site"]
        for k, (t, r, s) in enumerate(gpu["logs"]):
            lo = k * w.W
            hi = min((k + 1) * w.W, w.t_end)
            sel = (t_all >= lo) & (t_all < hi)
            order = np.lexsort((t_all[sel], r_all[sel]))  # region, then time
            assert np.array_equal(t, t_all[sel][order]), f"window {k} times"
            assert np.array_equal(r, r_all[sel][order]), f"window {k} regions"
            assert np.array_equal(s, s_all[sel][order]), f"window {k} sites"
    return ref, gpu
