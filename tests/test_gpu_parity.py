"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle,
bit-exact -- final spins, per-region event counts, per-region digests of the
full (fp64 time bits, site) sequences, and the per-window event logs.

Tolerance: none.  Both sides implement the same IEEE operation sequence
(DESIGN.md §3), so every fp64 event time must agree to the bit.
"""
import math

import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_cs_0405053_b200 import FLAG_DIGEST, FLAG_LOG_EVENTS, IsingSR, IsingSRError  # noqa: E402
from _gpu_common import check_against_oracle, run_gpu  # noqa: E402


def test_c1_bit_exact_full():
    """BASELINE config 1 in full: 16x16, 4x4 regions, T=1.5, W=1, t=10."""
    w = workloads.get("c1")
    ref, gpu = check_against_oracle(w)
    assert ref["n_events"] > 300
    assert max(gpu["g"]) >= 2  # real relaxation happened


@pytest.mark.parametrize("geom", [
    # Lx, Ly, bx, by, T, H, W, t_end, init
    (16, 16, 1, 1, 2.269, 0.0, 0.5, 4.0, "random"),
    (16, 16, 2, 2, 1.5, 0.0, 1.0, 6.0, "random"),
    (24, 16, 4, 4, 4.0, 0.3, 0.25, 3.0, "random"),
    (32, 32, 8, 8, 2.269, 0.0, 0.375, 8.0, "up"),
    (16, 24, 4, 8, 2.0, -0.2, 0.7, 5.0, "random"),
    (24, 16, 8, 4, 3.0, 0.0, 1.3, 5.0, "random"),
    (12, 20, 4, 2, 1.8, 0.1, 0.5, 6.0, "random"),
    (20, 12, 2, 4, 2.5, 0.0, 0.9, 6.0, "random"),
    (9, 9, 1, 1, 1.2, 0.0, 2.0, 10.0, "random"),
    (3, 3, 1, 1, 2.0, 0.0, 1.0, 30.0, "random"),
])
def test_geometries_bit_exact(geom):
    Lx, Ly, bx, by, T, H, W, t_end, init = geom
    w = workloads.Workload("g", Lx, Ly, bx, by, T=T, H=H, W=W, t_end=t_end, init=init, seed=7)
    check_against_oracle(w)


@pytest.mark.parametrize("geom", [(8, 8, 8, 8), (4, 4, 4, 4), (16, 8, 4, 8), (8, 16, 8, 4), (8, 4, 8, 4)])
def test_regions_spanning_a_dimension(geom):
    """Regions covering the lattice height and/or width wrap inside the region
    (no ghost on that axis); one region covering the lattice has g == 1."""
    Lx, Ly, bx, by = geom
    w = workloads.Workload("span", Lx, Ly, bx, by, T=2.0, W=0.8, t_end=6.0, seed=3)
    ref, gpu = check_against_oracle(w)
    if Lx == bx and Ly == by:
        assert set(gpu["g"]) == {1}


def test_single_region_equals_single_stream_bkl():
    w = workloads.Workload("one", 8, 8, 8, 8, T=2.269, W=1.0, t_end=10.0, seed=5)
    gpu = run_gpu(w, per_window_logs=True)
    b = oracle.bkl_run(8, 8, w.rates(), 5, w.spins(), 10.0, log_cap=10**6)
    t = np.concatenate([l[0] for l in gpu["logs"]])
    s = np.concatenate([l[2] for l in gpu["logs"]])
    assert np.array_equal(t, b["log_t"]) and np.array_equal(s, b["log_site"])


def test_c2_full_bit_exact():
    """BASELINE config 2 in full: 256^2, 8x8 regions, T=2.269, all up, W=0.375, t=100."""
    w = workloads.get("c2")
    check_against_oracle(w, logs=False)


@pytest.mark.parametrize("W", [0.25, 1.0, 4.0, 2.125, 0.1])
def test_window_invariance(W):
    """The fixed point does not depend on W (windows only schedule work)."""
    w = workloads.Workload("wi", 32, 32, 4, 4, T=2.0, W=W, t_end=8.0, seed=11)
    check_against_oracle(w, logs=False)


def test_capacity_overflow_retry_is_exact():
    w = workloads.Workload("cap", 32, 32, 4, 4, T=4.0, W=2.0, t_end=6.0, seed=2)
    gpu = run_gpu(w, per_window_logs=False, hist_capacity=1)
    assert gpu["stats"]["overflow_retries"] >= 1
    check_against_oracle(w, gpu=gpu, logs=False)


def test_diverged_window_is_not_committed():
    w = workloads.Workload("div", 32, 32, 2, 2, T=2.0, W=4.0, t_end=8.0, seed=4)
    sim = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.spins(), w.W, w.t_end, w.seed, max_iterations=2)
    with pytest.raises(IsingSRError) as e:
        sim.run_window()
    assert e.value.status == -4
    with pytest.raises(IsingSRError) as e:
        sim.commit()
    assert e.value.status == -9
    assert np.array_equal(sim.spins(), w.spins())  # committed state untouched
    st = sim.stats()
    assert st["windows"] == 0 and st["events_total"] == 0
    sim.close()


def test_determinism_and_idempotence():
    w = workloads.Workload("det", 64, 64, 4, 4, T=2.269, W=0.6, t_end=3.0, seed=8)
    a = run_gpu(w)
    b = run_gpu(w)
    assert a["g"] == b["g"]
    assert np.array_equal(a["digest"], b["digest"])
    # re-running an uncommitted window gives the same fixed point and g
    sim = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.spins(), w.W, w.t_end, w.seed)
    g1 = sim.run_window()
    g2 = sim.run_window()
    assert g1 == g2 == a["g"][0]
    sim.commit()
    sim.close()


def test_c4_full_lattice_across_a_window_boundary():
    """BASELINE config 4 at full size over t < 0.52: the first window [0, 0.5)
    with its full relaxation, its commit, and the start of the second window
    -- the bench's launch configuration -- against the oracle, region by
    region (about 3 minutes, mostly the serial oracle)."""
    w = workloads.get("c4", t_end=0.52)
    ref = oracle.des_workload(w)
    gpu = run_gpu(w, flags=FLAG_DIGEST)
    assert len(gpu["g"]) == 2 and gpu["events"] == ref["n_events"] > 5 * 10**7
    assert np.array_equal(gpu["count"], ref["count"])
    assert np.array_equal(gpu["digest"], ref["digest"])
    assert np.array_equal(gpu["spins"], ref["spins"])


def test_c4_full_lattice_prefix():
    """BASELINE config 4 at its full size (16384^2, 4x4 regions, T=2, W=0.5) on
    the prefix t < 0.02: every region's digest and count, and all spins."""
    w = workloads.get("c4", t_end=0.02)
    ref = oracle.des_workload(w)
    gpu = run_gpu(w, flags=FLAG_DIGEST)
    assert gpu["events"] == ref["n_events"] > 10**6
    assert np.array_equal(gpu["count"], ref["count"])
    assert np.array_equal(gpu["digest"], ref["digest"])
    assert np.array_equal(gpu["spins"], ref["spins"])


# ---------------------------------------------------------------------------
# warp-per-region form (regions of more than 64 sites: c3 16x16, c5 32x32)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("geom", [
    # Lx, Ly, bx, by, T, H, W, t_end, init
    (64, 64, 16, 16, 2.269, 0.0, 0.5, 3.0, "random"),
    (64, 64, 32, 32, 4.0, 0.0, 1.0, 3.0, "random"),
    (96, 64, 32, 32, 2.269, 0.0, 4.0, 8.0, "random"),
    (64, 96, 16, 32, 1.0, 0.1, 2.0, 10.0, "random"),
    (96, 48, 32, 16, 3.0, -0.2, 0.7, 4.0, "random"),
    (32, 48, 16, 8, 2.0, 0.0, 0.6, 5.0, "random"),
    (48, 32, 8, 16, 2.0, 0.0, 0.6, 5.0, "random"),
    (32, 32, 32, 32, 2.0, 0.0, 1.0, 6.0, "random"),   # one region: wraps both ways, g == 1
    (64, 32, 32, 32, 2.0, 0.0, 1.0, 6.0, "random"),   # two regions per row: W and E neighbour coincide
])
def test_warp_form_bit_exact(geom):
    Lx, Ly, bx, by, T, H, W, t_end, init = geom
    w = workloads.Workload("w", Lx, Ly, bx, by, T=T, H=H, W=W, t_end=t_end, init=init, seed=5)
    ref, gpu = check_against_oracle(w)
    if Lx == bx and Ly == by:
        assert set(gpu["g"]) == {1}


def test_c3_prefix_bit_exact():
    """BASELINE config 3 at full size (4096^2, 16x16 regions, T=1, H=0.1,
    W=2) on the prefix t < 4 (the bulk of its events)."""
    w = workloads.get("c3", t_end=4.0)
    check_against_oracle(w, logs=False)


def test_c5_geometry_sample_bit_exact():
    """c5 dynamics (H=0, 32x32 regions, T in {1, 2.269, 4}, W in {.25,1,4})
    on a 512^2 lattice."""
    for T in (1.0, 2.269, 4.0):
        for W in (0.25, 4.0):
            w = workloads.Workload("c5s", 512, 512, 32, 32, T=T, W=W, t_end=4.0, seed=1)
            check_against_oracle(w, logs=False)


# ---------------------------------------------------------------------------
# every schedule of K1 (lane-persistent with the pipelined host loop:
# default; one iteration per host sync: ISING_SR_PIPELINE=0; the warp form of
# big regions: ISING_SR_BIG=0; big regions without resume: ISING_SR_RESUME=0;
# the general K1 instantiation where the PLAIN one applies: ISING_SR_PLAIN=0)
# and an extreme refill threshold give the oracle's bits
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("env", [
    {},
    {"ISING_SR_PLAIN": "0"},
    {"ISING_SR_PIPELINE": "0"},
    {"ISING_SR_PIPELINE": "0", "ISING_SR_BIG": "0"},
    {"ISING_SR_REFILL": "1"},
    {"ISING_SR_BIG": "0"},
    {"ISING_SR_RESUME": "0"},
])
def test_k1_schedules_bit_exact(env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    check_against_oracle(workloads.get("c1"))
    for Lx, Ly, bx, by, T, W in [(64, 64, 4, 4, 2.0, 0.5), (32, 32, 8, 8, 2.269, 1.0), (16, 16, 1, 1, 2.0, 0.5),
                                 (24, 24, 2, 2, 1.5, 2.0), (64, 64, 16, 16, 2.269, 1.0), (64, 64, 32, 32, 4.0, 0.5)]:
        w = workloads.Workload("sched", Lx, Ly, bx, by, T=T, W=W, t_end=4.0, seed=9)
        check_against_oracle(w, logs=False)


# ---------------------------------------------------------------------------
# small worklists spread to one region per 2^k lanes (both lane-per-region
# kernels): lattices whose worklists pass through every k on
# the way down (n 2^k <= one wave), with the spread off, capped and full
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("env", [{}, {"ISING_SR_LANE_SPREAD": "0", "ISING_SR_BIG_SPREAD": "0"},
                                 {"ISING_SR_LANE_SPREAD": "2", "ISING_SR_BIG_SPREAD": "2"},
                                 {"ISING_SR_PIPELINE": "0"}, {"ISING_SR_GRAPH": "1"}])
def test_small_worklist_spread_bit_exact(env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    for Lx, Ly, bx, by, T, W, t_end in [(512, 512, 4, 4, 2.0, 0.5, 1.5), (512, 512, 2, 2, 2.269, 0.5, 1.0),
                                        (512, 256, 8, 8, 2.269, 1.0, 2.0), (512, 512, 16, 16, 2.269, 1.0, 2.0),
                                        (128, 128, 1, 1, 1.0, 0.5, 1.0)]:
        w = workloads.Workload("spread", Lx, Ly, bx, by, T=T, W=W, t_end=t_end, seed=21)
        check_against_oracle(w, logs=False)


@pytest.mark.parametrize("b,T,t_end", [(8, 2.269, 0.05), (32, 4.0, 0.05), (2, 1.0, 0.02)])
def test_c5_full_lattice_prefix(b, T, t_end):
    """c5 at its full size (8192^2) for b x b regions on a prefix of the run:
    every region's event count and digest, and all spins."""
    w = workloads.Workload(f"c5_b{b}", 8192, 8192, b, b, T=T, W=0.25, t_end=t_end, seed=1)
    ref = oracle.des_workload(w)
    gpu = run_gpu(w, flags=FLAG_DIGEST)
    assert gpu["events"] == ref["n_events"] > 10**5
    assert np.array_equal(gpu["count"], ref["count"])
    assert np.array_equal(gpu["digest"], ref["digest"])
    assert np.array_equal(gpu["spins"], ref["spins"])


# ---------------------------------------------------------------------------
# the alternate approach to subsequent steps: every window starts
# afresh with random numbers of a new generation; the oracle implements the
# same rule (fresh_W), every K1 form must match it bit for bit
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("geom", [
    (32, 32, 4, 4, 2.269, 0.5, 4.0),
    (16, 16, 1, 1, 2.0, 0.3, 2.0),
    (64, 64, 8, 8, 1.5, 0.7, 4.0),
    (64, 64, 16, 16, 2.269, 1.0, 4.0),
    (64, 64, 32, 32, 4.0, 0.25, 2.0),
])
@pytest.mark.parametrize("env", [{}, {"ISING_SR_BIG": "0"}])
def test_fresh_window_variant_bit_exact(geom, env, monkeypatch):
    from paper_cs_0405053_b200 import FLAG_FRESH_WINDOW
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    Lx, Ly, bx, by, T, W, t_end = geom
    w = workloads.Workload("fw", Lx, Ly, bx, by, T=T, W=W, t_end=t_end, seed=4)
    ref = oracle.des_workload(w, fresh_W=W)
    gpu = run_gpu(w, flags=FLAG_DIGEST | FLAG_FRESH_WINDOW)
    assert gpu["events"] == ref["n_events"]
    assert np.array_equal(gpu["count"], ref["count"])
    assert np.array_equal(gpu["spins"], ref["spins"])
    assert np.array_equal(gpu["digest"], ref["digest"])
    base = oracle.des_workload(w)
    assert not np.array_equal(base["digest"], ref["digest"])  # the variant changes the trajectory


def test_checkpoint_resume_bit_exact():
    """A run checkpointed at a committed time and resumed in a fresh ctx is
    bit-identical to the uninterrupted run; a corrupted checkpoint or one of
    another configuration is refused."""
    from paper_cs_0405053_b200 import FLAG_FRESH_WINDOW, FLAG_OBSERVABLES
    for flags in (FLAG_DIGEST, FLAG_DIGEST | FLAG_FRESH_WINDOW | FLAG_OBSERVABLES):
        w = workloads.Workload("ck", 64, 64, 4, 4, T=2.269, W=0.5, t_end=4.0, seed=6)
        full = run_gpu(w, flags=flags)
        a = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.spins(), w.W, w.t_end, w.seed, flags=flags)
        for _ in range(3):
            a.run_window()
            a.commit()
        ck = a.checkpoint()
        a.close()
        b = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.spins(), w.W, w.t_end, w.seed, flags=flags)
        b.restore(ck)
        ev = 0
        while True:
            try:
                b.run_window()
            except IsingSRError as e:
                assert e.status == -9
                break
            ev += b.commit()
        dig, cnt = b.digests()
        assert np.array_equal(dig, full["digest"]) and np.array_equal(cnt, full["count"])
        assert np.array_equal(b.spins(), full["spins"])
        assert b.stats()["events_total"] == full["events"]
        assert b.stats()["obs_B_total"] == full["stats"]["obs_B_total"]  # same windows, same sums
        bad = bytearray(ck)
        bad[-1] ^= 1
        with pytest.raises(IsingSRError):
            b.restore(bytes(bad))
        b.close()
        other = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.spins(), w.W, w.t_end, w.seed + 1, flags=flags)
        with pytest.raises(IsingSRError):
            other.restore(ck)
        other.close()


# ---------------------------------------------------------------------------
# FLAG_OBSERVABLES: per-region time integrals of M and of the bond sum B,
# reduced at commit.  Against the oracle's integrals of the global M(t), B(t)
# (different summation order: relative 1e-9), and against Onsager's exact
# energy and spontaneous magnetisation (an independent physics pin).
# ---------------------------------------------------------------------------
def _run_obs(w, **kw):
    from paper_cs_0405053_b200 import FLAG_OBSERVABLES
    sim = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.spins(), w.W, w.t_end, w.seed,
                  flags=FLAG_DIGEST | FLAG_OBSERVABLES, **kw)
    sim.run()
    st = sim.stats()
    dig, cnt = sim.digests()
    sim.close()
    return st, dig


@pytest.mark.parametrize("geom", [
    (32, 32, 4, 4, 2.269, 0.0, 0.5, 4.0),
    (24, 24, 2, 2, 1.8, 0.2, 0.7, 3.0),
    (16, 16, 1, 1, 3.0, 0.0, 0.4, 2.0),
    (32, 32, 8, 8, 2.0, 0.0, 0.6, 4.0),
    (64, 64, 16, 16, 2.269, 0.0, 1.0, 3.0),
    (32, 32, 32, 32, 2.5, 0.0, 0.8, 3.0),   # region = lattice: wrap bonds
    (32, 64, 32, 16, 2.0, 0.1, 0.5, 3.0),
    (12, 8, 4, 8, 2.0, 0.0, 0.5, 3.0),      # 4x8 regions spanning the height
])
def test_observables_against_oracle(geom):
    Lx, Ly, bx, by, T, H, W, t_end = geom
    w = workloads.Workload("obs", Lx, Ly, bx, by, T=T, H=H, W=W, t_end=t_end, seed=2)
    st, dig = _run_obs(w)
    ref = oracle.des_workload(w)
    dt, Bi, Mi = ref["obs"][0], ref["obs"][1], ref["obs"][2]
    assert np.array_equal(dig, ref["digest"])
    assert st["obs_time_total"] == pytest.approx(dt, rel=1e-12)
    scale = Lx * Ly * t_end
    assert abs(st["obs_M_total"] - Mi) < 1e-9 * scale, (st["obs_M_total"], Mi)
    assert abs(st["obs_B_total"] - Bi) < 1e-9 * scale, (st["obs_B_total"], Bi)


def test_observables_onsager():
    """256^2 at T = 2 from all up: time averages over t in [20, 60) of the
    energy per site and |m| against Onsager's exact values (finite-size
    corrections are far below the tolerance at correlation length ~2)."""
    from scipy.special import ellipk
    T = 2.0
    beta = 1.0 / T
    k = 2 * math.sinh(2 * beta) / math.cosh(2 * beta) ** 2
    u = -1 / math.tanh(2 * beta) * (1 + 2 / math.pi * (2 * math.tanh(2 * beta) ** 2 - 1) * ellipk(k * k))
    m0 = (1 - math.sinh(2 * beta) ** -4) ** 0.125
    from paper_cs_0405053_b200 import FLAG_OBSERVABLES
    w = workloads.Workload("ons", 256, 256, 4, 4, T=T, W=0.5, t_end=60.0, init="up", seed=3)
    sim = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.spins(), w.W, w.t_end, w.seed, flags=FLAG_OBSERVABLES)
    for _ in range(40):
        sim.run_window()
        sim.commit()
    a = sim.stats()
    absm, es = [], []
    while sim.stats()["t_c"] < w.t_end:
        sim.run_window()
        sim.commit()
        st = sim.stats()
        absm.append(abs(st["obs_M_now"]) / 65536)
        es.append(-st["obs_B_now"] / 65536)
    b = sim.stats()
    sim.close()
    n = 256 * 256
    # snapshots at the 80 committed times: |M| (not a time integral) and E
    assert abs(np.mean(absm) - m0) < 0.01, (np.mean(absm), m0)
    assert abs(np.mean(es) - u) < 0.006, (np.mean(es), u)
    tt = b["obs_time_total"] - a["obs_time_total"]
    e = -(b["obs_B_total"] - a["obs_B_total"]) / (n * tt)   # J = 1, H = 0
    m = (b["obs_M_total"] - a["obs_M_total"]) / (n * tt)
    assert tt == pytest.approx(40.0)
    assert abs(e - u) < 0.004, (e, u)
    assert abs(m - m0) < 0.01, (m, m0)


@pytest.mark.parametrize("env", [{}, {"ISING_SR_PIPELINE": "0"}])
def test_stats_active_regions_per_iteration(env, monkeypatch):
    """stats.active_last: the worklist length of every iteration of the last
    window -- all regions in iteration 1, the window's recomputations in
    total, nothing after iteration g; commit time is accounted."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    w = workloads.Workload("act", 64, 64, 4, 4, T=2.0, W=0.5, t_end=3.0, seed=5)
    sim = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.spins(), w.W, w.t_end, w.seed)
    nreg = (w.Lx // w.bx) * (w.Ly // w.by)
    prev = sim.stats()["recomputations_total"]
    for _ in range(4):
        sim.run_window()
        sim.commit()
        st = sim.stats()
        a = st["active_last"]
        assert a[0] == nreg
        assert sum(a) == st["recomputations_total"] - prev
        assert all(x == 0 for x in a[st["g_last"]:]) and all(x > 0 for x in a[:st["g_last"] - 1])
        prev = st["recomputations_total"]
    assert sim.stats()["ms_commit_total"] > 0.0
    sim.close()


@pytest.mark.parametrize("geom", [(64, 64, 4, 4, 2.0, 0.5), (64, 64, 16, 16, 2.269, 1.0), (32, 32, 2, 2, 1.5, 0.7)])
def test_jacobi_all_same_fixed_point_and_g(geom):
    """FLAG_JACOBI_ALL (every region in every iteration, the paper's schedule):
    the oracle's bits, and per window the same g as the worklist schedule,
    with g x N recomputations."""
    from paper_cs_0405053_b200 import FLAG_JACOBI_ALL
    Lx, Ly, bx, by, T, W = geom
    w = workloads.Workload("jac", Lx, Ly, bx, by, T=T, W=W, t_end=4.0, seed=8)
    nreg = (Lx // bx) * (Ly // by)
    a = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.spins(), w.W, w.t_end, w.seed, flags=FLAG_DIGEST)
    b = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.spins(), w.W, w.t_end, w.seed,
                flags=FLAG_DIGEST | FLAG_JACOBI_ALL)
    r0 = 0
    for _ in range(w.n_windows()):
        ga, gb = a.run_window(), b.run_window()
        assert ga == gb
        a.commit()
        b.commit()
        r1 = b.stats()["recomputations_total"]
        assert r1 - r0 == gb * nreg
        r0 = r1
    ref = oracle.des_workload(w)
    da, ca = a.digests()
    db, cb = b.digests()
    assert np.array_equal(db, da) and np.array_equal(cb, ca)
    assert np.array_equal(cb, ref["count"])
    assert np.array_equal(db, ref["digest"])
    assert np.array_equal(b.spins(), ref["spins"])
    a.close()
    b.close()


def test_torch_caching_allocator_hooks():
    """dev_alloc/dev_free hooks (torch's caching allocator): every device
    buffer is torch's, results are the oracle's, including a capacity-overflow
    retry that reallocates the histories; all returned on close."""
    import torch
    torch.cuda.synchronize()
    m0 = torch.cuda.memory_allocated()
    w = workloads.Workload("cap", 32, 32, 4, 4, T=4.0, W=2.0, t_end=6.0, seed=2)
    sim = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.spins(), w.W, w.t_end, w.seed, hist_capacity=1,
                  torch_alloc=True)
    assert torch.cuda.memory_allocated() > m0
    sim.run()
    st = sim.stats()
    assert st["overflow_retries"] >= 1
    dig, cnt = sim.digests()
    spins = sim.spins()
    sim.close()
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated() == m0
    ref = oracle.des_workload(w)
    assert np.array_equal(cnt, ref["count"]) and np.array_equal(dig, ref["digest"])
    assert np.array_equal(spins, ref["spins"])


@pytest.mark.parametrize("geom", [(64, 64, 4, 4), (8, 24, 8, 4), (64, 64, 16, 16), (32, 64, 32, 32), (24, 8, 8, 8), (64, 16, 16, 16)])
def test_observables_snapshot_at_committed_times(geom):
    """stats.obs_M_now / obs_B_now: M and the bond sum of the configuration at
    every committed time, against a direct count on the returned spins
    (lane and big regions, regions spanning the lattice width)."""
    from paper_cs_0405053_b200 import FLAG_OBSERVABLES
    Lx, Ly, bx, by = geom
    w = workloads.Workload("snap", Lx, Ly, bx, by, T=2.269, W=0.5, t_end=2.0, seed=6)
    sim = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.spins(), w.W, w.t_end, w.seed, flags=FLAG_OBSERVABLES)

    def direct():
        s = sim.spins().reshape(Ly, Lx).astype(np.int64) * 2 - 1
        return int(s.sum()), int((s * np.roll(s, -1, 0)).sum() + (s * np.roll(s, -1, 1)).sum())

    for _ in range(w.n_windows()):
        st = sim.stats()
        assert (st["obs_M_now"], st["obs_B_now"]) == direct()
        sim.run_window()
        sim.commit()
    st = sim.stats()
    assert (st["obs_M_now"], st["obs_B_now"]) == direct()
    sim.close()


# ---------------------------------------------------------------------------
# the device-side window loop (ISING_SR_GRAPH=1: one CUDA graph per window,
# iteration 1 + a conditional while node of two iterations per trip, the
# decision taken on the device): same bits and the same g per window as the
# host loops, incl. a capacity-overflow restart and divergence
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("geom", [(64, 64, 4, 4, 2.0, 0.5), (32, 32, 8, 8, 2.269, 1.0), (16, 16, 1, 1, 2.0, 0.5),
                                  (64, 64, 16, 16, 2.269, 1.0), (64, 64, 32, 32, 4.0, 0.5)])
def test_device_window_loop_bit_exact(geom, monkeypatch):
    Lx, Ly, bx, by, T, W = geom
    w = workloads.Workload("graph", Lx, Ly, bx, by, T=T, W=W, t_end=4.0, seed=9)
    host = run_gpu(w)
    monkeypatch.setenv("ISING_SR_GRAPH", "1")
    ref, dev = check_against_oracle(w)
    assert dev["g"] == host["g"]
    assert dev["stats"]["recomputations_total"] == host["stats"]["recomputations_total"]
    assert dev["stats"]["region_ms"] > 0.0


def test_device_window_loop_overflow_and_divergence(monkeypatch):
    monkeypatch.setenv("ISING_SR_GRAPH", "1")
    w = workloads.Workload("cap", 32, 32, 4, 4, T=4.0, W=2.0, t_end=6.0, seed=2)
    gpu = run_gpu(w, per_window_logs=False, hist_capacity=1)
    assert gpu["stats"]["overflow_retries"] >= 1
    check_against_oracle(w, gpu=gpu, logs=False)
    w = workloads.Workload("div", 32, 32, 2, 2, T=2.0, W=4.0, t_end=8.0, seed=4)
    sim = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.spins(), w.W, w.t_end, w.seed, max_iterations=2)
    with pytest.raises(IsingSRError) as e:
        sim.run_window()
    assert e.value.status == -4
    assert np.array_equal(sim.spins(), w.spins())
    sim.close()
