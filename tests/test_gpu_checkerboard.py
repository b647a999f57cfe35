"""Second workload on the GPU: checkerboard Metropolis
sweeps (ising_cb_run / ising_cb_sweeps) against the pinned oracle
(orc_cb_run) bit for bit -- every spin and the accepted-flip count -- on
both kernel forms (word form when Lx % 4 == 0, site form otherwise), ragged
sizes, offsets, a split run, the full c4 lattice, degenerate tables; and in
distribution against Onsager's exact energy and magnetisation (the same
equilibrium as the n-fold way's, test_observables_onsager)."""
import math

import numpy as np
import pytest
import torch

import oracle
import workloads
from paper_cs_0405053_b200 import IsingSRError, checkerboard_run, checkerboard_sweeps

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("Lx,Ly,T,H,rule,seed,sweep0,n", [
    (64, 64, 2.269, 0.0, "metropolis", 1, 0, 10),      # word form
    (130, 66, 2.0, 0.0, "metropolis", 2, 0, 7),        # site form (Lx % 4 == 2), ragged against the block
    (4, 4, 1.5, 0.0, "metropolis", 3, 0, 25),          # smallest lattice
    (12, 8, 3.0, 0.4, "glauber", 4, 5, 9),             # field, Glauber, sweep offset
    (1000, 6, 4.0, -0.3, "metropolis", 5, 2**33 + 7, 3),  # 64-bit sweep counter
    (6, 1002, 1.0, 0.1, "glauber", 6, 0, 4),           # tall, site form
])
def test_cb_bit_exact(Lx, Ly, T, H, rule, seed, sweep0, n):
    p = workloads.rate_table(T, 1.0, H, rule)
    s0 = workloads.initial_spins(Lx, Ly, "random", seed)
    ref, rf = oracle.cb_run(s0, Lx, Ly, p, seed, sweep0, n)
    got, gf = checkerboard_run(s0, Lx, Ly, p, seed, sweep0, n)
    assert gf == rf > 0
    assert np.array_equal(got, ref)


def test_cb_degenerate_tables_and_zero_sweeps():
    s0 = workloads.initial_spins(16, 8, "random", 1)
    got, f = checkerboard_run(s0, 16, 8, [1.0] * 10, 9, 0, 1)
    assert f == 128 and np.array_equal(got, 1 - s0.reshape(-1))
    got, f = checkerboard_run(s0, 16, 8, [0.0] * 10, 9, 0, 5)
    assert f == 0 and np.array_equal(got, s0.reshape(-1))
    got, f = checkerboard_run(s0, 16, 8, [0.5] * 10, 9, 0, 0)
    assert f == 0 and np.array_equal(got, s0.reshape(-1))


def test_cb_invalid_arguments():
    with pytest.raises(IsingSRError):
        checkerboard_run(np.zeros(25, np.uint8), 5, 5, [0.5] * 10, 1, 0, 1)
    with pytest.raises(IsingSRError):
        checkerboard_run(np.zeros(16, np.uint8), 4, 4, [2.0] + [0.5] * 9, 1, 0, 1)
    with pytest.raises(IsingSRError):
        checkerboard_run(np.zeros(16, np.uint8), 4, 4, [0.5] * 10, 1, -1, 1)
    with pytest.raises(IsingSRError):
        checkerboard_run(np.zeros(16, np.uint8), 4, 4, [0.5] * 10, 1, 2**62, 1)  # the colour bit of the counter


def test_cb_device_api_split_run():
    """Device-resident lattice, the run split at sweep 3: identical to the
    oracle's run in one piece; flips accumulate in a device counter."""
    Lx, Ly, seed = 256, 128, 7
    p = workloads.rate_table(2.269)
    s0 = workloads.initial_spins(Lx, Ly, "random", seed)
    ref, rf = oracle.cb_run(s0, Lx, Ly, p, seed, 0, 8)
    d = torch.from_numpy(s0.reshape(-1).copy()).cuda()
    fl = torch.zeros(1, dtype=torch.int64, device="cuda")
    checkerboard_sweeps(d.data_ptr(), Lx, Ly, p, seed, 0, 3, fl.data_ptr())
    checkerboard_sweeps(d.data_ptr(), Lx, Ly, p, seed, 3, 5, fl.data_ptr())
    torch.cuda.synchronize()
    assert int(fl.item()) == rf
    assert np.array_equal(d.cpu().numpy(), ref)


def test_cb_full_c4_lattice():
    """The c4 lattice (16384^2, T = 2, seed 1), two sweeps: every spin."""
    w = workloads.get("c4")
    p = w.rates()
    s0 = w.spins()
    ref, rf = oracle.cb_run(s0, w.Lx, w.Ly, p, w.seed, 0, 2)
    got, gf = checkerboard_run(s0, w.Lx, w.Ly, p, w.seed, 0, 2)
    assert gf == rf > 10**8
    assert np.array_equal(got, ref)


def test_cb_onsager():
    """256^2 at T = 2 from all up, sweeps 500..3499: the sweep averages of the
    energy per site and |m| against Onsager's exact values."""
    from scipy.special import ellipk
    T = 2.0
    beta = 1.0 / T
    k = 2 * math.sinh(2 * beta) / math.cosh(2 * beta) ** 2
    u = -1 / math.tanh(2 * beta) * (1 + 2 / math.pi * (2 * math.tanh(2 * beta) ** 2 - 1) * ellipk(k * k))
    m0 = (1 - math.sinh(2 * beta) ** -4) ** 0.125
    L = 256
    p = workloads.rate_table(T)
    d = torch.ones(L * L, dtype=torch.uint8, device="cuda")
    checkerboard_sweeps(d.data_ptr(), L, L, p, 3, 0, 500)
    es, ms = [], []
    for s in range(500, 3500, 10):
        checkerboard_sweeps(d.data_ptr(), L, L, p, 3, s, 10)
        sp = d.view(L, L).to(torch.int32) * 2 - 1
        B = (sp * torch.roll(sp, -1, 0)).sum() + (sp * torch.roll(sp, -1, 1)).sum()
        es.append(-B.item() / (L * L))
        ms.append(abs(sp.sum().item()) / (L * L))
    assert abs(np.mean(es) - u) < 0.004, (np.mean(es), u)
    assert abs(np.mean(ms) - m0) < 0.01, (np.mean(ms), m0)
