"""GPU parity of the round-2 features, against the CPU oracle bit for bit:
exact time ties (quantized budgets), Glauber rates on the n-fold-way path,
the commit-time compaction of K1's event log (including forced replays) and
the h count of SURVEY §8(d.3), the device-generated initial spins, and the
paper's window T_max = ln N / (lambda |dG|)."""
import math

import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_cs_0405053_b200 import FLAG_DIGEST, FLAG_LOG_EVENTS, IsingSR  # noqa: E402
from _gpu_common import check_against_oracle, run_gpu  # noqa: E402


def _ties(ref):
    """(events sharing their time with an event of another region, clamped
    budgets are not visible here) in the oracle's global log."""
    t, r = ref["log_t"], ref["log_region"]
    order = np.lexsort((r, t))
    ts, rs = t[order], r[order]
    same = (ts[1:] == ts[:-1]) & (rs[1:] != rs[:-1])
    return int(same.sum())


# ---------------------------------------------------------------------------
# tie mode (R30): budgets (floor(E q) + 1) / q with q = 4 make exact
# time ties between regions common; the (time, region id) order (R10) and the
# candidate bump (R11) decide them identically on both sides
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("geom", [
    # Lx, Ly, bx, by, T, W, t_end
    (32, 32, 4, 4, math.inf, 0.5, 3.0),
    (16, 16, 1, 1, math.inf, 0.25, 2.0),
    (24, 24, 2, 2, math.inf, 0.7, 3.0),
    (32, 32, 8, 8, math.inf, 0.5, 2.0),
    (32, 32, 4, 4, 2.269, 0.5, 4.0),
    (64, 64, 16, 16, math.inf, 0.5, 1.5),
    (64, 64, 32, 32, math.inf, 0.5, 1.0),
])
def test_tie_mode_bit_exact(geom):
    Lx, Ly, bx, by, T, W, t_end = geom
    w = workloads.Workload("tie", Lx, Ly, bx, by, T=T, W=W, t_end=t_end, seed=3)
    ref, gpu = check_against_oracle(w, oracle_kw={"eq_quantum": 4.0}, eq_quantum=4.0)
    assert _ties(ref) > (10 if math.isinf(T) else 2), "the mode must produce exact ties across regions"
    if math.isinf(T) and bx == 4:  # budgets clamped to 0 by a tied break point: candidates bumped (R11)
        assert ref["n_bumps"] > 0
    assert gpu["events"] > 0


def test_tie_mode_oracle_order_is_time_then_region():
    """The oracle's processing order in the tie mode is the lexicographic
    (time, region id) order (readings R10/R11); many events tie."""
    w = workloads.Workload("tie", 32, 32, 4, 4, T=math.inf, W=1.0, t_end=2.0, seed=5)
    ref = oracle.des_workload(w, log_cap=10**6, eq_quantum=4.0)
    t, r = ref["log_t"], ref["log_region"]
    assert np.all((t[1:] > t[:-1]) | ((t[1:] == t[:-1]) & (r[1:] > r[:-1])))
    assert _ties(ref) > 50


# ---------------------------------------------------------------------------
# Glauber rates (eq. pglauber) with H != 0: all ten class rates
# distinct, on every K1 form
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("geom", [
    (32, 32, 4, 4, 0.5, 4.0), (16, 16, 1, 1, 0.5, 3.0), (24, 24, 2, 2, 0.7, 4.0), (32, 32, 8, 8, 0.5, 4.0),
    (24, 16, 8, 4, 0.6, 4.0), (64, 64, 16, 16, 1.0, 3.0), (64, 64, 32, 32, 0.5, 2.0),
])
def test_glauber_rates_bit_exact(geom):
    Lx, Ly, bx, by, W, t_end = geom
    w = workloads.Workload("gl", Lx, Ly, bx, by, T=1.7, H=0.3, W=W, t_end=t_end, seed=12, rule="glauber")
    r = w.rates()
    assert len(set(r)) == 10 and max(r) < 1.0
    check_against_oracle(w)


# ---------------------------------------------------------------------------
# K3: the commit compacts the events K1 recorded in each region's final
# recomputation; regions with more than log_capacity events are replayed.
# The logs equal the oracle's window by window for any capacity, and
# stats.edge_entries_last_window is the number of (event, region edge it
# lies on) pairs -- h of SURVEY §8(d.3) -- of the window's committed events
# ---------------------------------------------------------------------------
def _edge_entries(t, site, lo, hi, bx, by, wrapx, wrapy):
    sel = (t >= lo) & (t < hi)
    s = site[sel].astype(np.int64)
    sr, sc = s // bx, s % bx
    n = 0
    if not wrapy:
        n += int((sr == 0).sum()) + int((sr == by - 1).sum())
    if not wrapx:
        n += int((sc == 0).sum()) + int((sc == bx - 1).sum())
    return n


@pytest.mark.parametrize("cap", [0, 1, 3])
@pytest.mark.parametrize("geom", [(32, 32, 4, 4, 2.0, 0.5), (24, 24, 2, 2, 1.5, 1.0), (32, 32, 8, 8, 2.269, 0.5),
                                  (16, 16, 1, 1, 2.0, 0.5), (64, 64, 16, 16, 2.269, 1.0), (8, 16, 8, 4, 2.0, 0.5)])
def test_log_compaction_and_edge_entries(geom, cap):
    Lx, Ly, bx, by, T, W = geom
    w = workloads.Workload("log", Lx, Ly, bx, by, T=T, W=W, t_end=3.0, seed=21)
    ref, gpu = check_against_oracle(w, log_capacity=cap)
    for k, st in enumerate(gpu["window_stats"]):
        lo, hi = k * W, min((k + 1) * W, w.t_end)
        want = _edge_entries(ref["log_t"], ref["log_site"], lo, hi, bx, by, Lx == bx, Ly == by)
        assert st["edge_entries_last_window"] == want, k
        if cap == 1:
            n_multi = np.count_nonzero(np.bincount(gpu["logs"][k][1], minlength=1) > 1)
            assert st["log_replayed_last_window"] == n_multi, k


# ---------------------------------------------------------------------------
# initial spins generated on the device from the Philox init stream (SURVEY
# §8(c.3)) equal the input generator's (workloads.initial_spins), including a
# seed with a nonzero high word and strips of a multi-rank run
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("geom", [(48, 40, 4, 4, 1), (36, 12, 2, 2, 0x123456789), (64, 64, 16, 16, 7),
                                  (16384, 16384, 4, 4, 1)])
def test_device_initial_spins(geom):
    Lx, Ly, bx, by, seed = geom
    want = workloads.initial_spins(Lx, Ly, "random", seed)
    rates = workloads.rate_table(2.0)
    sim = IsingSR(Lx, Ly, bx, by, rates, None, 0.5, 1.0, seed)
    got = sim.spins()
    sim.close()
    assert np.array_equal(got, want)
    if Ly // by % 2 == 0 and Lx * Ly <= 1 << 16:
        for q in range(2):
            s = IsingSR(Lx, Ly, bx, by, rates, None, 0.5, 1.0, seed, rank=q, world=2)
            n = Lx * Ly // 2
            assert np.array_equal(s.spins(), want[q * n:(q + 1) * n])
            s.close()


def test_device_initial_spins_run_equals_host_spins_run():
    """A run started from device-generated spins is the run started from the
    same configuration passed from the host."""
    w = workloads.Workload("dev", 64, 64, 4, 4, T=2.269, W=0.5, t_end=3.0, seed=9)
    a = run_gpu(w)
    sim = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), None, w.W, w.t_end, w.seed)
    sim.run()
    dig, cnt = sim.digests()
    spins = sim.spins()
    sim.close()
    assert np.array_equal(dig, a["digest"]) and np.array_equal(cnt, a["count"])
    assert np.array_equal(spins, a["spins"])


# ---------------------------------------------------------------------------
# the paper's window T_max = ln N / (lambda |dG_i|), |dG_i| =
# boundary sites of a region (4b - 4; 1 for 1x1): any W gives the same
# trajectory, and with W = T_max the relaxation converges
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("b", [1, 2, 4, 8, 16])
def test_paper_window_tmax(b):
    L = 64
    N = (L // b) ** 2
    dG = 1 if b == 1 else 4 * b - 4
    W = workloads.paper_tmax(N, dG)
    assert W == pytest.approx(math.log(N) / dG)
    w = workloads.Workload("tmax", L, L, b, b, T=2.269, W=W, t_end=2.0, seed=4)
    ref, gpu = check_against_oracle(w, logs=False)
    assert len(gpu["g"]) == w.n_windows()
    # W <= 0 in the C ABI selects the same rule (lambda = the largest rate)
    sim = IsingSR(L, L, b, b, w.rates(), w.spins(), 0.0, 2.0, 4)
    sim.run_window()
    sim.commit()
    assert sim.stats()["t_c"] == min(W, 2.0)
    sim.close()


# ---------------------------------------------------------------------------
# FLAG_MAG_MOMENTS: int |M| dt and int M^2 dt per
# window from the device time sort of the committed log, against the
# oracle's integrals over the global M(t) (ising_oracle.c obs[3], obs[4];
# only the summation order differs: relative 1e-9), on lane and big regions
# and with forced replays; and the time average of |M| against Onsager's m0
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("geom", [
    (32, 32, 4, 4, 2.269, 0.0, 0.5, 4.0, 0), (24, 24, 2, 2, 1.8, 0.2, 0.7, 3.0, 0), (16, 16, 1, 1, 3.0, 0.0, 0.4, 2.0, 0),
    (32, 32, 8, 8, 2.0, 0.0, 0.6, 4.0, 0), (64, 64, 16, 16, 2.269, 0.0, 1.0, 3.0, 0), (32, 32, 4, 4, 2.0, 0.1, 0.5, 3.0, 1),
])
def test_magnetisation_moments_against_oracle(geom):
    from paper_cs_0405053_b200 import FLAG_MAG_MOMENTS
    Lx, Ly, bx, by, T, H, W, t_end, cap = geom
    w = workloads.Workload("mm", Lx, Ly, bx, by, T=T, H=H, W=W, t_end=t_end, seed=2)
    sim = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.spins(), w.W, w.t_end, w.seed,
                  flags=FLAG_DIGEST | FLAG_MAG_MOMENTS, log_capacity=cap)
    sim.run()
    st = sim.stats()
    dig, _ = sim.digests()
    sim.close()
    ref = oracle.des_workload(w)
    assert np.array_equal(dig, ref["digest"])
    scale1 = Lx * Ly * t_end
    assert abs(st["obs_absM_total"] - ref["obs"][3]) < 1e-9 * scale1, (st["obs_absM_total"], ref["obs"][3])
    assert abs(st["obs_M2_total"] - ref["obs"][4]) < 1e-9 * scale1 * Lx * Ly, (st["obs_M2_total"], ref["obs"][4])
    assert abs(st["obs_M_total"] - ref["obs"][2]) < 1e-9 * scale1


def test_magnetisation_moments_onsager():
    """256^2 at T = 2 from all up: the time average of |m| over t in [20, 60)
    against Onsager's spontaneous magnetisation (correlation length ~2)."""
    from paper_cs_0405053_b200 import FLAG_MAG_MOMENTS
    T = 2.0
    m0 = (1 - math.sinh(2 / T) ** -4) ** 0.125
    w = workloads.Workload("ons", 256, 256, 4, 4, T=T, W=0.5, t_end=60.0, init="up", seed=3)
    sim = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.spins(), w.W, w.t_end, w.seed, flags=FLAG_MAG_MOMENTS)
    for _ in range(40):
        sim.run_window()
        sim.commit()
    a = sim.stats()
    sim.run()
    b = sim.stats()
    sim.close()
    n = 256 * 256
    tt = b["obs_time_total"] - a["obs_time_total"]
    absm = (b["obs_absM_total"] - a["obs_absM_total"]) / (n * tt)
    m2 = (b["obs_M2_total"] - a["obs_M2_total"]) / (n * n * tt)
    assert tt == pytest.approx(40.0)
    assert abs(absm - m0) < 0.01, (absm, m0)
    assert m2 >= absm ** 2 - 1e-12  # <m^2> >= <|m|>^2
    assert abs(math.sqrt(m2) - m0) < 0.012
