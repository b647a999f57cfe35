"""Pins for the oracle's primitives (CPU only).

Each test pins one oracle function to something other than itself:
published known-answer vectors, an independent implementation (ATen),
libm, or a closed form.
"""
import math
import os
import shutil
import subprocess

import numpy as np
import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))


def _kat():
    rows = []
    with open(os.path.join(HERE, "golden", "philox4x32_10_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            v = [int(x, 16) for x in line.split()]
            rows.append((v[:4], v[4:6], tuple(v[6:10])))
    return rows


def test_philox_known_answer_vectors():
    # Random123 KAT vectors (tests/golden/philox4x32_10_kat.txt)
    for ctr, key, want in _kat():
        assert oracle.philox(ctr, key) == want


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_philox_matches_aten_engine(tmp_path):
    """Independent implementation: ATen's host philox_engine."""
    import torch
    inc = os.path.join(os.path.dirname(torch.__file__), "include")
    exe = tmp_path / "pa"
    subprocess.check_call(["g++", "-O1", "-std=c++17", "-I" + inc, "-o", str(exe),
                           os.path.join(HERE, "philox_aten_check.cpp")])
    rng = np.random.default_rng(7)
    ctr = rng.integers(0, 2**32, size=(2000, 4), dtype=np.uint64).astype(np.uint32)
    key = rng.integers(0, 2**32, size=(2000, 2), dtype=np.uint64).astype(np.uint32)
    # include structured counters as used by the method: (n, 0, 0, seed_hi)
    ctr[:100, 1:] = 0
    ctr[:100, 0] = np.arange(100)
    lines = "\n".join(" ".join(f"{int(x):x}" for x in list(c) + list(k)) for c, k in zip(ctr, key))
    out = subprocess.run([str(exe)], input=lines, capture_output=True, text=True, check=True).stdout
    ref = np.array([[int(x, 16) for x in l.split()] for l in out.strip().splitlines()], dtype=np.uint32)
    got = oracle.philox_n(ctr, key)
    assert np.array_equal(got, ref)


def test_pair_mapping_exact_and_in_range():
    """U, V = ((x_hi<<32 | x_lo) >> 12 + 0.5) * 2^-52 from the Philox words of
    key = (stream, seed_lo), counter = (n_lo, n_hi, 0, seed_hi)."""
    seed = 0x0123456789ABCDEF
    streams = np.arange(50, dtype=np.uint32).repeat(20)
    idx = np.tile(np.arange(20, dtype=np.uint64), 50) + np.uint64(2**32 - 5)
    U, V = oracle.pair_n(seed, streams, idx)
    ctr = np.zeros((streams.shape[0], 4), dtype=np.uint32)
    ctr[:, 0] = (idx & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    ctr[:, 1] = (idx >> np.uint64(32)).astype(np.uint32)
    ctr[:, 3] = seed >> 32
    key = np.zeros((streams.shape[0], 2), dtype=np.uint32)
    key[:, 0] = streams
    key[:, 1] = seed & 0xFFFFFFFF
    x = oracle.philox_n(ctr, key).astype(np.uint64)
    a = ((x[:, 0] << np.uint64(32)) | x[:, 1]) >> np.uint64(12)
    b = ((x[:, 2] << np.uint64(32)) | x[:, 3]) >> np.uint64(12)
    # exact: U * 2^52 - 0.5 is the integer a
    assert np.array_equal(U * 2.0**52 - 0.5, a.astype(np.float64))
    assert np.array_equal(V * 2.0**52 - 0.5, b.astype(np.float64))
    assert (U >= 2.0**-53).all() and (U <= 1 - 2.0**-53).all()
    assert (V > 0).all() and (V < 1).all()


def _ulp_diff(a, b):
    ia = a.view(np.int64)
    ib = b.view(np.int64)
    return np.abs(ia - ib)


def test_expvar_vs_libm_random():
    """E(U) = -log U within 4 ulp of libm over 2e6 uniform U (eq. nextau)."""
    rng = np.random.default_rng(3)
    a = rng.integers(0, 2**52, size=2_000_000, dtype=np.uint64)
    U = (a.astype(np.float64) + 0.5) * 2.0**-52
    E = oracle.expvar_n(U)
    ref = -np.log(U)
    assert (E > 0).all()
    assert _ulp_diff(E, ref).max() <= 4


def test_expvar_edge_values():
    vals = [2.0**-53, 1 - 2.0**-53, 0.5, 0.25, 2.0**-20, 1 - 2.0**-30,
            math.sqrt(2) / 2, np.nextafter(math.sqrt(2) / 2, 0), np.nextafter(math.sqrt(2) / 2, 1),
            0.75, 1e-10, 0.999999]
    U = np.array(vals, dtype=np.float64)
    E = oracle.expvar_n(U)
    ref = -np.log(U)
    assert (E > 0).all()
    assert _ulp_diff(E, ref).max() <= 4
    # closed forms: -log(2^-k) = k ln 2 (to within the ln2 split's rounding)
    for k in (1, 2, 20, 53):
        assert abs(oracle.expvar(2.0**-k) - k * math.log(2)) <= 2 * np.spacing(k * math.log(2))


def test_expvar_mean_is_one():
    """E(U) of uniform U is Exp(1): mean 1, variance 1."""
    U, _ = oracle.pair_n(11, np.zeros(400_000, np.uint32), np.arange(400_000, dtype=np.uint64))
    E = oracle.expvar_n(U)
    assert abs(E.mean() - 1) < 5 / math.sqrt(400_000)
    assert abs(E.var() - 1) < 10 / math.sqrt(400_000)


def test_mix64_is_splitmix64_finalizer():
    # splitmix64 with state 0 returns mix(0x9e3779b97f4a7c15) = 0xe220a8397b1dcdaf
    # as its first output (Steele, Lea, Flood, OOPSLA 2014; java.util.SplittableRandom)
    assert oracle.mix64(0x9E3779B97F4A7C15) == 0xE220A8397B1DCDAF
    assert oracle.mix64(0) == 0


def test_candidate_time_closed_forms():
    # eq. nextau: tau = tau_prev + E/Lambda (Lambda=2, E=1 -> 0.5)
    assert oracle.cand(0.0, 1.0, 2.0) == 0.5
    # Lambda = 0: no event
    assert math.isinf(oracle.cand(3.0, 1.0, 0.0))
    # rounding onto itself bumps to the next double (reading #11)
    t = 1.0e6
    assert oracle.cand(t, 1e-30, 1.0) == np.nextafter(t, np.inf)
    assert oracle.cand(0.0, 0.0, 1.0) == np.nextafter(0.0, 1.0)


def test_breakpoint_integration_closed_form():
    """eqs. lambdataua/breaksum/bsubk/newtau: Lambda = 1 on (0,1),
    then 3, with -log U = 2: int_0^tau Lambda = 2 -> tau = 1 + 1/3."""
    R = oracle.breakpoint_budget(2.0, 1.0, 1.0, 0.0)
    assert R == 1.0
    assert oracle.cand(1.0, R, 3.0) == 1.0 + 1.0 / 3.0
    # budget exhausted before the break point: clamp at 0 (reading #11)
    assert oracle.breakpoint_budget(0.5, 1.0, 1.0, 0.0) == 0.0


def test_breakpoint_integration_vs_bisection():
    """Random piecewise-constant Lambda profiles: solving eq. lambdataua by
    successive break points equals bisection on the integral."""
    rng = np.random.default_rng(5)
    for _ in range(2000):
        nb = rng.integers(0, 6)
        tb = np.sort(rng.uniform(0, 3, size=nb))
        lam = rng.uniform(0.1, 5, size=nb + 1)
        E = rng.exponential()
        t_s, R, seg = 0.0, E, 0
        tau = oracle.cand(t_s, R, lam[0])
        while seg < nb and tb[seg] < tau:
            R = oracle.breakpoint_budget(R, lam[seg], tb[seg], t_s)
            t_s = tb[seg]
            seg += 1
            tau = oracle.cand(t_s, R, lam[seg])

        def integral(t):
            edges = np.concatenate([[0.0], tb, [np.inf]])
            s = 0.0
            for i in range(nb + 1):
                a, b = edges[i], min(edges[i + 1], t)
                if b > a:
                    s += lam[i] * (b - a)
            return s
        lo, hi = 0.0, 1e3
        for _ in range(200):
            mid = 0.5 * (lo + hi)
            if integral(mid) < E:
                lo = mid
            else:
                hi = mid
        assert abs(tau - lo) <= 1e-9 * max(1.0, lo)


def test_fold_and_selection_examples():
    rates = [0.5, 0.25, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 0.25, 0.5]
    N = [2, 0, 3, 0, 0, 0, 0, 0, 1, 4]
    lam = oracle.fold(N, rates)
    assert lam == 2 * 0.5 + 3 * 1.0 + 1 * 0.25 + 4 * 0.5
    # brute force: the class k* and index j of x = V*Lambda
    rng = np.random.default_rng(1)
    cum = np.cumsum([n * r for n, r in zip(N, rates)])
    for V in rng.uniform(0, 1, size=5000):
        k, j = oracle.select(N, rates, V, lam)
        x = V * lam
        k_ref = int(np.searchsorted(cum, x, side="left"))
        assert k == k_ref
        below = cum[k - 1] if k > 0 else 0.0
        assert j == min(int(math.floor((x - below) / rates[k])), N[k] - 1)
        assert 0 <= j < N[k]
    # SPEC S:262-263 in x-space: weights (1,3); x exactly at the boundary picks
    # the first class, beyond it the second
    r2 = [1.0] + [0.0] * 9
    r2[1] = 3.0
    N2 = [1, 1] + [0] * 8
    assert oracle.select(N2, r2, 0.25, 4.0)[0] == 0
    assert oracle.select(N2, r2, np.nextafter(0.25, 1), 4.0)[0] == 1
    # clamp of eq. vindex when V = W(k) exactly (reading #8)
    assert oracle.select([4] + [0] * 9, [1.0] * 10, 1 - 2.0**-53, 4.0) == (0, 3)


def test_selection_frequencies_proportional_to_rates():
    """Phase 2 picks class k with probability N_k r_k / Lambda (eq. Wsum)."""
    rates = [0.1, 0.3, 1.0, 1.0, 1.0, 1.0, 1.0, 0.7, 0.2, 0.05]
    N = [3, 1, 2, 0, 5, 1, 0, 2, 4, 7]
    lam = oracle.fold(N, rates)
    U, V = oracle.pair_n(9, np.zeros(100_000, np.uint32), np.arange(100_000, dtype=np.uint64))
    counts = np.zeros(10)
    for v in V[:100_000]:
        counts[oracle.select(N, rates, v, lam)[0]] += 1
    p = np.array([n * r for n, r in zip(N, rates)]) / lam
    exp = p * 100_000
    for k in range(10):
        assert abs(counts[k] - exp[k]) <= 5 * math.sqrt(exp[k] + 1)
