"""Pins for the input generator (problem statement) and the oracle's
classification, against SPEC.md worked examples and brute force."""
import json
import math
import os

import numpy as np

import oracle
import workloads

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "spec_examples.json")))


def _energy(spins, Lx, Ly, J, H):
    s = (2 * spins.astype(np.int64) - 1).reshape(Ly, Lx)
    B = (s * np.roll(s, -1, 0)).sum() + (s * np.roll(s, -1, 1)).sum()
    return -J * B - H * s.sum()


def test_delta_energy_examples():
    for ex in GOLD["delta_energy"]:
        k = 5 * (ex["s"] + 1) // 2 + (ex["sigma"] + 4) // 2
        assert workloads.delta_energy(k, ex["J"], ex["H"]) == ex["dE"], ex["cite"]


def test_delta_energy_matches_brute_force():
    """dE = 2 J s sigma + 2 H s equals E(after) - E(before) of eq. hamil."""
    rng = np.random.default_rng(0)
    for _ in range(300):
        Lx, Ly = rng.integers(3, 7, size=2)
        J, H = rng.uniform(0.2, 2), rng.uniform(-1, 1)
        s = rng.integers(0, 2, size=Lx * Ly).astype(np.uint8)
        v = rng.integers(0, Lx * Ly)
        y, x = divmod(v, Lx)
        g = s.reshape(Ly, Lx)
        u = int(g[(y - 1) % Ly, x] + g[(y + 1) % Ly, x] + g[y, (x - 1) % Lx] + g[y, (x + 1) % Lx])
        k = 5 * int(s[v]) + u
        t = s.copy()
        t[v] ^= 1
        ref = _energy(t, Lx, Ly, J, H) - _energy(s, Lx, Ly, J, H)
        assert abs(workloads.delta_energy(k, J, H) - ref) <= 1e-12 * max(1, abs(ref))


def test_total_energy_examples():
    for ex in GOLD["total_energy"]:
        s = workloads.initial_spins(ex["Lx"], ex["Ly"], ex["init"])
        assert _energy(s, ex["Lx"], ex["Ly"], ex["J"], ex["H"]) == ex["E"], ex["cite"]


def test_class_code_examples():
    for ex in GOLD["class_code"]:
        k = 5 * (ex["s"] + 1) // 2 + ex["u"]
        assert k == ex["k"]
        assert workloads.class_spin(k) == ex["s"] and workloads.class_up(k) == ex["u"]


def test_rate_table_examples_and_closed_forms():
    for ex in GOLD["flip_probability"]:
        r = workloads.rate_table(ex["T"], ex["J"], ex["H"], ex["rule"])
        assert abs(r[ex["k"]] - ex["p"]) <= 1e-15, ex["cite"]
    # H = 0 Metropolis: [e^-8/T, e^-4/T, 1,1,1,1,1,1, e^-4/T, e^-8/T]
    for T in (1.0, 1.5, 2.0, 2.269, 4.0):
        r = workloads.rate_table(T)
        want = [math.exp(-8 / T), math.exp(-4 / T)] + [1.0] * 6 + [math.exp(-4 / T), math.exp(-8 / T)]
        assert r == want
    r = workloads.rate_table(float("inf"))
    assert r == [1.0] * 10
    # Glauber detailed balance: p(dE)/p(-dE) = exp(-dE/T)
    T, H = 1.7, 0.3
    g = workloads.rate_table(T, 1.0, H, "glauber")
    for k in range(10):
        dE = workloads.delta_energy(k, 1.0, H)
        # the reverse move of class k: flipped spin with same neighbours
        kr = (k + 5) % 10
        assert abs(g[k] / g[kr] - math.exp(-dE / T)) < 1e-12
        assert g[k] < 1


def test_class_count_examples():
    for ex in GOLD["class_counts"]:
        s = workloads.initial_spins(ex["Lx"], ex["Ly"], ex["init"])
        if "flip" in ex:
            s[ex["flip"]] ^= 1
        N = oracle.class_counts(ex["Lx"], ex["Ly"], ex["Lx"], ex["Ly"], s)[0]
        want = np.zeros(10, dtype=np.int32)
        for k, n in ex["N"].items():
            want[int(k)] = n
        assert np.array_equal(N, want), ex["cite"]


def test_class_counts_brute_force_per_region():
    rng = np.random.default_rng(2)
    for (Lx, Ly, bx, by) in [(8, 8, 2, 2), (12, 6, 4, 3), (5, 7, 1, 1), (16, 16, 16, 4)]:
        s = rng.integers(0, 2, size=Lx * Ly).astype(np.uint8)
        N = oracle.class_counts(Lx, Ly, bx, by, s)
        g = s.reshape(Ly, Lx).astype(int)
        u = np.roll(g, 1, 0) + np.roll(g, -1, 0) + np.roll(g, 1, 1) + np.roll(g, -1, 1)
        k = 5 * g + u
        RX = Lx // bx
        ref = np.zeros_like(N)
        for y in range(Ly):
            for x in range(Lx):
                ref[(y // by) * RX + x // bx, k[y, x]] += 1
        assert np.array_equal(N, ref)


def test_initial_spins_deterministic_and_balanced():
    a = workloads.initial_spins(256, 256, "random", seed=1)
    b = workloads.initial_spins(256, 256, "random", seed=1)
    c = workloads.initial_spins(256, 256, "random", seed=2)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    assert abs(a.mean() - 0.5) < 5 * 0.5 / 256
    assert set(np.unique(a)) <= {0, 1}


def test_config_presets_match_baseline_json():
    c = workloads.CONFIGS
    assert (c["c1"].Lx, c["c1"].bx, c["c1"].T, c["c1"].W, c["c1"].t_end) == (16, 4, 1.5, 1.0, 10.0)
    assert (c["c2"].Lx, c["c2"].bx, c["c2"].T, c["c2"].init) == (256, 8, 2.269, "up")
    assert (c["c3"].Lx, c["c3"].bx, c["c3"].H, c["c3"].W, c["c3"].t_end) == (4096, 16, 0.1, 2.0, 200.0)
    assert (c["c4"].Lx, c["c4"].bx, c["c4"].T, c["c4"].W, c["c4"].t_end) == (16384, 4, 2.0, 0.5, 50.0)
    assert c["c4"].n_regions == 16_777_216
    assert len(workloads.c5_points()) == 45
    # exact initial rate per site of c1 / c4 (rounded)
    assert abs(workloads.exact_initial_rate_per_site(c["c1"]) - 0.705) < 0.05


def _kat_rows():
    rows = []
    for line in open(os.path.join(HERE, "golden", "philox4x32_10_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(x, 16) for x in line.split()]
        rows.append((v[:4], v[4:6], v[6:10]))
    return rows


def test_init_stream_philox_kat():
    """The input generator's Philox4x32-10 reproduces the Random123 known-answer
    vectors (tests/golden/philox4x32_10_kat.txt)."""
    for ctr, key, out in _kat_rows():
        got = workloads.philox4x32_10(np.array([ctr], dtype=np.uint32), np.array([key], dtype=np.uint32))
        assert [int(x) for x in got[0]] == out


def test_init_stream_layout_against_oracle_philox():
    """SURVEY §8(c.3) init stream: site v is bit (v & 31) of word ((v >> 5) & 3)
    of Philox(key=(0xFFFFFFFF, seed_lo), ctr=(v >> 7, 0, 1, seed_hi)), checked
    site by site with the oracle's independent Philox on a 37x29 lattice (a
    ragged last draw) and two seeds (one with a nonzero high word)."""
    for seed in (1, 0x123456789):
        Lx, Ly = 37, 29
        s = workloads.initial_spins(Lx, Ly, "random", seed)
        for v in range(Lx * Ly):
            w = oracle.philox([v >> 7, 0, 1, seed >> 32], [0xFFFFFFFF, seed & 0xFFFFFFFF])
            assert s[v] == (w[(v >> 5) & 3] >> (v & 31)) & 1, (seed, v)


def test_init_stream_statistics():
    """iid p = 1/2: the up fraction and nearest-neighbour correlation of a
    1024^2 draw are within 5 sigma of 1/2 and 0."""
    s = workloads.initial_spins(1024, 1024, "random", 1).astype(np.float64)
    n = s.size
    assert abs(s.mean() - 0.5) < 5 * 0.5 / math.sqrt(n)
    g = 2 * s.reshape(1024, 1024) - 1
    assert abs((g * np.roll(g, 1, 1)).mean()) < 5 / math.sqrt(n)
    assert abs((g * np.roll(g, 1, 0)).mean()) < 5 / math.sqrt(n)
