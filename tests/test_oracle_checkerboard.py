"""Pins of the checkerboard Metropolis oracle (orc_cb_run; SURVEY §8f row 4:
the discrete-time dynamics of the paper's §2) against what the
mathematics fixes, independent of the oracle's own code:

* p = 1 for every class: every visited atom flips, so one sweep inverts the
  lattice (closed form);
* p = 0: nothing moves;
* the chain's stationary distribution is the Boltzmann distribution of
  eq. hamil for Metropolis and Glauber rates (each colour pass
  is a product of single-site updates that satisfy detailed balance):
  long-run sweep averages of E, |M| and M on 4x4 against exact enumeration
  over all 2^16 states -- a wrong class index, sign or neighbour fails;
* a run split in two (sweep0 offset) equals the run in one piece, and the
  visiting order within a colour does not matter (the same sweep computed
  with the colours' sites processed in a different order, by a brute-force
  reference that decides each site with the oracle's pinned Philox draw).
"""
import numpy as np
import pytest

import oracle
import workloads
from oracle.exact import boltzmann_averages


def energy_mag(s, Lx, Ly, J=1.0, H=0.0):
    sp = (2 * s.astype(np.int64) - 1).reshape(Ly, Lx)
    B = (sp * np.roll(sp, -1, 0)).sum() + (sp * np.roll(sp, -1, 1)).sum()
    M = sp.sum()
    return -J * B - H * M, M


def test_p_one_inverts_every_sweep():
    s0 = workloads.initial_spins(8, 6, "random", 3)
    s1, f1 = oracle.cb_run(s0, 8, 6, [1.0] * 10, 5, 0, 1)
    assert np.array_equal(s1, 1 - s0.reshape(-1)) and f1 == 48
    s3, f3 = oracle.cb_run(s0, 8, 6, [1.0] * 10, 5, 0, 3)
    assert np.array_equal(s3, 1 - s0.reshape(-1)) and f3 == 3 * 48


def test_p_zero_is_frozen():
    s0 = workloads.initial_spins(10, 4, "random", 7)
    s, f = oracle.cb_run(s0, 10, 4, [0.0] * 10, 5, 0, 20)
    assert np.array_equal(s, s0.reshape(-1)) and f == 0


def test_invalid_arguments():
    s0 = np.zeros(25, np.uint8)
    with pytest.raises(ValueError):
        oracle.cb_run(s0, 5, 5, [0.5] * 10, 1, 0, 1)  # odd: not bipartite
    with pytest.raises(ValueError):
        oracle.cb_run(np.zeros(16, np.uint8), 4, 4, [1.5] + [0.5] * 9, 1, 0, 1)


def test_split_run_equals_one_run():
    s0 = workloads.initial_spins(12, 8, "random", 2)
    p = workloads.rate_table(2.269)
    a, fa = oracle.cb_run(s0, 12, 8, p, 9, 0, 7)
    b1, f1 = oracle.cb_run(s0, 12, 8, p, 9, 0, 3)
    b2, f2 = oracle.cb_run(b1, 12, 8, p, 9, 3, 4)
    assert np.array_equal(a, b2) and fa == f1 + f2


def _philox_u(Lx, y, x, colour, s, seed):
    j = x // 2
    q = y * ((Lx + 2) // 4) + j // 2
    w = oracle.philox([q, s & 0xFFFFFFFF, (s >> 32) | (colour << 31), seed >> 32], [0xFFFFFFFE, seed & 0xFFFFFFFF])
    hi, lo = (w[2], w[3]) if j % 2 else (w[0], w[1])
    a = ((int(hi) << 32) | int(lo)) >> 12
    return (a + 0.5) * 2.0 ** -52


@pytest.mark.parametrize("Lx,Ly", [(6, 4), (8, 6)])  # Lx % 4 == 2: the last site of a row and colour draws alone
def test_any_order_within_a_colour(Lx, Ly):
    """Brute force: visit each colour's sites in reverse (column-major,
    bottom-up) order, deciding every site with its pinned Philox draw."""
    seed = 11
    p = [0.05 * (k + 1) for k in range(10)]  # distinct per class: a wrong class index shows
    s0 = workloads.initial_spins(Lx, Ly, "random", 4).reshape(Ly, Lx).astype(np.int64)
    s = s0.copy()
    for sw in range(3):
        for colour in (0, 1):
            for x in reversed(range(Lx)):
                for y in reversed(range(Ly)):
                    if (x + y) % 2 != colour:
                        continue
                    u = s[(y - 1) % Ly, x] + s[(y + 1) % Ly, x] + s[y, (x - 1) % Lx] + s[y, (x + 1) % Lx]
                    k = 5 * s[y, x] + u
                    if _philox_u(Lx, y, x, colour, sw, seed) < p[k]:
                        s[y, x] ^= 1
    got, _ = oracle.cb_run(s0.astype(np.uint8), Lx, Ly, p, seed, 0, 3)
    assert np.array_equal(got, s.reshape(-1).astype(np.uint8))


@pytest.mark.parametrize("T,H,rule", [(2.5, 0.0, "metropolis"), (2.0, 0.3, "metropolis"), (3.0, -0.2, "glauber")])
def test_stationary_distribution_is_boltzmann(T, H, rule):
    Lx = Ly = 4
    p = workloads.rate_table(T, 1.0, H, rule)
    ex = boltzmann_averages(Lx, Ly, T, 1.0, H)
    s = workloads.initial_spins(Lx, Ly, "random", 1).reshape(-1)
    s, _ = oracle.cb_run(s, Lx, Ly, p, 21, 0, 200)  # burn-in
    nb, per = 100, 400
    Es, As, Ms = [], [], []
    sweep = 200
    for _ in range(nb):
        e = a = m = 0.0
        for _ in range(per):
            s, _ = oracle.cb_run(s, Lx, Ly, p, 21, sweep, 1)
            sweep += 1
            E, M = energy_mag(s, Lx, Ly, 1.0, H)
            e += E
            a += abs(M)
            m += M
        Es.append(e / per)
        As.append(a / per)
        Ms.append(m / per)
    for name, xs in (("E", Es), ("absM", As), ("M", Ms)):
        xs = np.array(xs)
        se = xs.std(ddof=1) / np.sqrt(nb)
        assert abs(xs.mean() - ex[name]) < 5 * se + 1e-9, (name, xs.mean(), ex[name], se)
