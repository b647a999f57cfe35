"""Pins for the whole oracle trajectory (CPU only).

* one region covering the lattice == the textbook single-stream n-fold way,
  bit for bit ("first iteration ... is almost a literal repetition
  of the sequential algorithm"; with one region there are no break points);
* integer-tracked energy/magnetisation and class counts equal a scratch
  recomputation after every event;
* exact Boltzmann averages by enumeration of all 2^9 states of 3x3
  (detailed balance of eq. pMin), for 1x1, 3x1 and 3x3 regions --
  1x1 regions make every event a break point for 4 regions (eqs.
  lambdataua..newtau), so a wrong budget update biases the averages;
* T = inf closed form E[m(t)] = m0 exp(-2t) and Poisson event counts;
* distributional agreement (KS) with the single-stream n-fold way.
"""
import math

import numpy as np
import pytest
from scipy import stats

import oracle
import workloads
from oracle.exact import boltzmann_averages


@pytest.mark.parametrize("L,T,seed", [(16, 1.5, 1), (8, 2.269, 5), (12, 4.0, 9), (5, 1.0, 3)])
def test_single_region_equals_single_stream_bkl(L, T, seed):
    rates = workloads.rate_table(T)
    s0 = workloads.initial_spins(L, L, "random", seed=seed)
    a = oracle.des_run(L, L, L, L, rates, seed, s0, 8.0, log_cap=10**6)
    b = oracle.bkl_run(L, L, rates, seed, s0, 8.0, stream=0, log_cap=10**6)
    assert a["n_events"] == b["n_events"] > 10
    assert np.array_equal(a["log_t"], b["log_t"])  # bit-exact fp64 event times
    assert np.array_equal(a["log_site"], b["log_site"])
    assert np.array_equal(a["spins"], b["spins"])
    assert a["digest"][0] == b["digest"][0]


def test_single_region_nonsquare_lattice_equals_bkl():
    rates = workloads.rate_table(2.0, 1.0, 0.2)
    s0 = workloads.initial_spins(7, 4, "random", seed=4)
    a = oracle.des_run(7, 4, 7, 4, rates, 4, s0, 20.0, log_cap=10**6)
    b = oracle.bkl_run(7, 4, rates, 4, s0, 20.0, log_cap=10**6)
    assert np.array_equal(a["log_t"], b["log_t"]) and np.array_equal(a["log_site"], b["log_site"])


@pytest.mark.parametrize("geom", [(8, 8, 4, 4), (6, 6, 1, 1), (8, 6, 2, 3), (9, 9, 3, 9), (16, 16, 4, 4)])
def test_incremental_invariants_after_every_event(geom):
    Lx, Ly, bx, by = geom
    rates = workloads.rate_table(3.0, 1.0, 0.3)
    s0 = workloads.initial_spins(Lx, Ly, "random", seed=2)
    r = oracle.des_run(Lx, Ly, bx, by, rates, 2, s0, 10.0, check=True)
    assert r["n_events"] > 50
    assert r["check_failures"] == 0
    # final (M, B) sample equals scratch recomputation
    r2 = oracle.des_run(Lx, Ly, bx, by, rates, 2, s0, 4.0, sample_t=[4.0])
    g = 2 * r2["spins"].astype(np.int64).reshape(Ly, Lx) - 1
    assert r2["sample_M"][0] == g.sum()
    assert r2["sample_B"][0] == (g * np.roll(g, -1, 0)).sum() + (g * np.roll(g, -1, 1)).sum()


def test_per_region_times_strictly_increase_and_order():
    w = workloads.get("c1")
    r = oracle.des_workload(w, log_cap=10**6)
    t, reg = r["log_t"], r["log_region"]
    # global processing order strictly increasing in (time, region id) (reading #10/#11)
    key_ok = (t[1:] > t[:-1]) | ((t[1:] == t[:-1]) & (reg[1:] > reg[:-1]))
    assert key_ok.all()
    for q in range(w.n_regions):
        tq = t[reg == q]
        assert (np.diff(tq) > 0).all()
    assert (t < w.t_end).all() and (t >= 0).all()
    assert int(r["count"].sum()) == r["n_events"]


@pytest.mark.parametrize("bx,by", [(1, 1), (3, 1), (3, 3)])
def test_boltzmann_3x3_time_averages(bx, by):
    T = 2.0
    ex = boltzmann_averages(3, 3, T)
    rates = workloads.rate_table(T)
    vals = {"E": [], "absM": [], "M2": []}
    for seed in range(1, 17):
        s0 = workloads.initial_spins(3, 3, "random", seed=seed)
        r = oracle.des_run(3, 3, bx, by, rates, seed, s0, 100000.0, t_obs0=20.0)
        dt, Bi, Mi, aMi, M2i = r["obs"]
        vals["E"].append(-Bi / dt)
        vals["absM"].append(aMi / dt)
        vals["M2"].append(M2i / dt)
    for q in vals:
        a = np.array(vals[q])
        se = a.std(ddof=1) / math.sqrt(len(a))
        assert abs(a.mean() - ex[q]) < 4 * se + 1e-9, (q, a.mean(), ex[q], se)


def test_boltzmann_3x3_with_field_and_glauber():
    T, H = 1.5, 0.4
    ex = boltzmann_averages(3, 3, T, 1.0, H)
    rates = workloads.rate_table(T, 1.0, H, "glauber")
    Es, Ms = [], []
    for seed in range(1, 17):
        s0 = workloads.initial_spins(3, 3, "random", seed=seed)
        r = oracle.des_run(3, 3, 1, 1, rates, seed, s0, 100000.0, t_obs0=20.0)
        dt, Bi, Mi, aMi, M2i = r["obs"]
        Es.append((-Bi - H * Mi) / dt)
        Ms.append(Mi / dt)
    for a, want in ((np.array(Es), ex["E"]), (np.array(Ms), ex["M"])):
        se = a.std(ddof=1) / math.sqrt(len(a))
        assert abs(a.mean() - want) < 4 * se


def test_infinite_temperature_closed_form():
    """All r_k = 1: every site flips as an independent rate-1 Poisson process,
    so E[m(t)] = m0 exp(-2t), Var[m(t)] = (1 - exp(-4t))/N, and the number of
    events in region i is Poisson(b^2 t)."""
    L, b = 64, 4
    N = L * L
    rates = [1.0] * 10
    ts = [0.1, 0.25, 0.5, 1.0]
    ms = []
    counts = []
    for seed in range(1, 9):
        s0 = workloads.initial_spins(L, L, "up")
        r = oracle.des_run(L, L, b, b, rates, seed, s0, 1.0, sample_t=ts)
        ms.append(r["sample_M"] / N)
        counts.append(r["count"])
    ms = np.array(ms)
    nseed = ms.shape[0]
    for i, t in enumerate(ts):
        sd = math.sqrt((1 - math.exp(-4 * t)) / N / nseed)
        assert abs(ms[:, i].mean() - math.exp(-2 * t)) < 4.5 * sd
        # variance across seeds consistent with (1-e^{-4t})/N (chi2, loose)
        var = ms[:, i].var(ddof=1)
        assert var < 4 * (1 - math.exp(-4 * t)) / N
    c = np.concatenate(counts).astype(np.float64)  # Poisson(16 * 1.0) per region
    assert abs(c.mean() - 16.0) < 4 * math.sqrt(16.0 / c.size)
    assert abs(c.var() - 16.0) < 0.1 * 16.0


def test_ks_against_single_stream_bkl():
    """Per-region streams and the single global stream give the same law of
    (M(t), E(t)) at fixed t."""
    L, b, T, t = 8, 2, 2.269, 1.5
    rates = workloads.rate_table(T)
    s0 = workloads.initial_spins(L, L, "random", seed=77)
    Md, Bd, Mb, Bb = [], [], [], []
    for seed in range(1, 601):
        r = oracle.des_run(L, L, b, b, rates, seed, s0, t, sample_t=[t])
        Md.append(r["sample_M"][0]); Bd.append(r["sample_B"][0])
        q = oracle.bkl_run(L, L, rates, seed + 100000, s0, t, sample_t=[t])
        Mb.append(q["sample_M"][0]); Bb.append(q["sample_B"][0])
    for a, c in ((Md, Mb), (Bd, Bb)):
        a, c = np.array(a, float), np.array(c, float)
        assert stats.ks_2samp(a, c).pvalue > 1e-3
        se = math.sqrt(a.var() / a.size + c.var() / c.size)
        assert abs(a.mean() - c.mean()) < 4 * se


def test_no_interaction_union_of_independent_runs():
    """Regions whose boundary sites cannot flip evolve independently: with
    rates zero for every class an all-up boundary frame can be in, each
    region's trajectory equals a one-region run of its own stream."""
    # all sites up except interior 2x2 blocks of each 4x4 region; rates: only
    # classes with s = down (k < 5) may flip, and only if u <= 3 (so an up
    # spin never flips: boundary sites of every region stay up).
    L, b = 12, 4
    s0 = np.ones((L, L), dtype=np.uint8)
    rng = np.random.default_rng(4)
    for ry in range(L // b):
        for rx in range(L // b):
            blk = rng.integers(0, 2, size=(2, 2))
            s0[ry * b + 1:ry * b + 3, rx * b + 1:rx * b + 3] = blk
    rates = [0.3, 0.5, 0.7, 0.9, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0]
    r = oracle.des_run(L, L, b, b, rates, 3, s0.reshape(-1), 50.0, log_cap=10**6)
    assert r["n_events"] > 0
    # each 4x4 region alone on a 4x4 periodic lattice sees the same (all-up)
    # frame, so its trajectory is the single-stream run of stream q
    for q in range(9):
        ry, rx = divmod(q, 3)
        blk = s0[ry * b:ry * b + b, rx * b:rx * b + b].reshape(-1)
        one = oracle.bkl_run(b, b, rates, 3, blk, 50.0, stream=q, log_cap=10**4)
        sel = r["log_region"] == q
        assert np.array_equal(r["log_t"][sel], one["log_t"])
        assert np.array_equal(r["log_site"][sel], one["log_site"])


# ---------------------------------------------------------------------------
# the alternate approach to subsequent steps: at every committed
# time t_c = w W every region discards its pending budget and starts afresh
# with random numbers of a new generation.  Unbiased by memorylessness of the
# Poisson process (the paper's claim), so the equilibrium and the T = inf
# relaxation are unchanged while the trajectory is not.
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("bx,by", [(1, 1), (3, 3)])
def test_fresh_window_boltzmann_3x3(bx, by):
    T = 2.0
    ex = boltzmann_averages(3, 3, T)
    rates = workloads.rate_table(T)
    vals = {"E": [], "absM": [], "M2": []}
    for seed in range(1, 17):
        s0 = workloads.initial_spins(3, 3, "random", seed=seed)
        r = oracle.des_run(3, 3, bx, by, rates, seed, s0, 50000.0, t_obs0=20.0, fresh_W=0.37)
        dt, Bi, Mi, aMi, M2i = r["obs"]
        vals["E"].append(-Bi / dt)
        vals["absM"].append(aMi / dt)
        vals["M2"].append(M2i / dt)
    for q in vals:
        a = np.array(vals[q])
        se = a.std(ddof=1) / math.sqrt(len(a))
        assert abs(a.mean() - ex[q]) < 4 * se + 1e-9, (q, a.mean(), ex[q], se)


def test_fresh_window_infinite_temperature_closed_form():
    L, b = 64, 4
    N = L * L
    ts = [0.1, 0.25, 0.5, 1.0]
    ms = []
    for seed in range(1, 9):
        s0 = workloads.initial_spins(L, L, "up")
        r = oracle.des_run(L, L, b, b, [1.0] * 10, seed, s0, 1.0, sample_t=ts, fresh_W=0.15)
        ms.append(r["sample_M"] / N)
    ms = np.array(ms)
    for i, t in enumerate(ts):
        sd = math.sqrt((1 - math.exp(-4 * t)) / N / ms.shape[0])
        assert abs(ms[:, i].mean() - math.exp(-2 * t)) < 4.5 * sd


def test_fresh_window_identity_and_effect():
    w = workloads.Workload("fw", 32, 32, 4, 4, T=2.269, W=0.5, t_end=3.0, seed=3)
    base = oracle.des_workload(w)
    # no committed time before t_end: nothing is wiped, bit-identical
    same = oracle.des_workload(w, fresh_W=5.0)
    assert np.array_equal(same["digest"], base["digest"]) and same["n_events"] == base["n_events"]
    # wiping at t_c = 0.5, 1.0, ... changes the trajectory
    fresh = oracle.des_workload(w, fresh_W=0.5)
    assert not np.array_equal(fresh["digest"], base["digest"])
    assert fresh["check_failures"] == 0


def test_tie_mode_exercises_the_candidate_bump():
    """Quantized budgets at T = inf (all rates 1): break points tied with a
    region's candidate clamp its budget to 0 and its next candidate is bumped
    to nextafter(t_s) (reading #11); with continuous budgets that never happens."""
    import math
    w = workloads.Workload("tie", 32, 32, 4, 4, T=math.inf, W=0.5, t_end=3.0, seed=3)
    assert oracle.des_workload(w, eq_quantum=4.0)["n_bumps"] > 0
    assert oracle.des_workload(w)["n_bumps"] == 0
