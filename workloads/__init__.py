"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic (no Philox event stream, no
exponential variates, no class logic, no event loop).  It only produces the
problem statement the paper starts from (§2):

* the lattice size, region size, J, H, T, window W and run length of each
  BASELINE.json config (c1..c5), and
* the initial spin configuration s(v), iid from the seeded
  Philox init stream, and
* the per-class flip-rate table r_k = lambda * p_k (eq. pMin /
  pglauber), computed ONCE here with libm exp and handed, as the same double
  bits, to both the oracle and the CUDA library (SURVEY §8c.3 "Rate table").

Both `oracle/` and `paper_cs_0405053_b200/` take these as inputs; neither
imports the other.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional

import numpy as np

# ---------------------------------------------------------------------------
# Rate table.  Class code k = 5*(s+1)/2 + u, where s is
# the atom's spin and u in 0..4 its number of up neighbours (class
# numbering per SURVEY §8c.4 #7).  sigma = sum of neighbour spins = 2u - 4.
# Delta E of flipping s -> -s under eq. hamil with each bond counted once
# (SURVEY §8c.4 #16): dE = 2 J s sigma + 2 H s.  lambda = 1 (reading #14).
# ---------------------------------------------------------------------------


def class_spin(k: int) -> int:
    return 1 if k >= 5 else -1


def class_up(k: int) -> int:
    return k % 5


def delta_energy(k: int, J: float, H: float) -> float:
    s = class_spin(k)
    sigma = 2 * class_up(k) - 4
    return 2.0 * J * s * sigma + 2.0 * H * s


def rate_table(T: float, J: float = 1.0, H: float = 0.0, rule: str = "metropolis",
               lam: float = 1.0) -> List[float]:
    """r_k = lambda * p_k.  Metropolis p = min(1, theta) (eq. pMin);
    Glauber p = theta/(1+theta) (eq. pglauber); theta = exp(-dE/T)
    with T meaning k_B T_abs in units of J (reading #15).  T = inf gives
    theta = 1 for every class."""
    out = []
    for k in range(10):
        dE = delta_energy(k, J, H)
        if math.isinf(T):
            theta = 1.0
        else:
            theta = math.exp(-dE / T)
        if rule == "metropolis":
            p = 1.0 if dE <= 0.0 else min(1.0, theta)
        elif rule == "glauber":
            p = theta / (1.0 + theta)
        else:
            raise ValueError(f"unknown rule {rule!r}")
        out.append(lam * p)
    return out


# ---------------------------------------------------------------------------
# Initial spins.  1 = up (+1), 0 = down (-1), row-major (row * Lx + col).
# "iid +-1 (p=0.5, seed s)" is the SURVEY §8(c.3) Philox init stream (reading
# #19): Philox4x32-10 with key = (0xFFFFFFFF, seed_lo), counter =
# (site >> 7, 0, 1, seed_hi); the spin of `site` is bit (site & 31) of output
# word ((site >> 5) & 3), 1 = up.  One draw gives 128 sites.  Key 0xFFFFFFFF
# is disjoint from the event-pair streams (key word 0 = region id < 2^31) and
# counter word 2 = 1 from their generation-0 counters.  The CUDA library
# implements the same counter-based generator independently (ising_sr_init
# with spins == NULL); the oracle never generates spins, it takes them as
# input.  Other p_up values use numpy's seeded Philox bit generator.
# ---------------------------------------------------------------------------

_PHILOX_M0, _PHILOX_M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
_PHILOX_W0, _PHILOX_W1 = 0x9E3779B9, 0xBB67AE85
_MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr: np.ndarray, key: np.ndarray) -> np.ndarray:
    """Vectorised Philox4x32-10 (Salmon et al., SC11): ctr (n, 4), key (n, 2)
    uint32 -> (n, 4) uint32.  Input generation only (pinned against the
    Random123 known-answer vectors in tests/test_workloads.py)."""
    c = [np.asarray(ctr, dtype=np.uint64)[:, i].copy() for i in range(4)]
    k0 = np.asarray(key, dtype=np.uint64)[:, 0].copy()
    k1 = np.asarray(key, dtype=np.uint64)[:, 1].copy()
    for r in range(10):
        if r:
            k0 = (k0 + np.uint64(_PHILOX_W0)) & _MASK32
            k1 = (k1 + np.uint64(_PHILOX_W1)) & _MASK32
        p0 = _PHILOX_M0 * c[0]
        p1 = _PHILOX_M1 * c[2]
        c = [(p1 >> np.uint64(32)) ^ c[1] ^ k0, p1 & _MASK32,
             (p0 >> np.uint64(32)) ^ c[3] ^ k1, p0 & _MASK32]
    return np.stack(c, axis=1).astype(np.uint32)


def philox_init_spins(Lx: int, Ly: int, seed: int = 1) -> np.ndarray:
    """iid +-1 spins (p = 1/2) from the Philox init stream (see above)."""
    n = Ly * Lx
    nd = (n + 127) // 128
    q = np.arange(nd, dtype=np.uint64)
    ctr = np.zeros((nd, 4), dtype=np.uint64)
    ctr[:, 0] = q & _MASK32
    ctr[:, 1] = q >> np.uint64(32)
    ctr[:, 2] = 1
    ctr[:, 3] = (seed >> 32) & 0xFFFFFFFF
    key = np.zeros((nd, 2), dtype=np.uint64)
    key[:, 0] = 0xFFFFFFFF
    key[:, 1] = seed & 0xFFFFFFFF
    out = philox4x32_10(ctr, key)                      # (nd, 4) words
    bits = np.unpackbits(out.astype("<u4").view(np.uint8), bitorder="little")
    return bits[:n].astype(np.uint8)                   # site = 128 q + 32 w + b


def initial_spins(Lx: int, Ly: int, init: str = "random", seed: int = 1,
                  p_up: float = 0.5) -> np.ndarray:
    if init == "up":
        return np.ones(Ly * Lx, dtype=np.uint8)
    if init == "down":
        return np.zeros(Ly * Lx, dtype=np.uint8)
    if init == "checker":
        yy, xx = np.meshgrid(np.arange(Ly), np.arange(Lx), indexing="ij")
        return ((yy + xx) % 2 == 0).astype(np.uint8).reshape(-1)
    if init == "random":
        if p_up == 0.5:
            return philox_init_spins(Lx, Ly, seed)
        g = np.random.Generator(np.random.Philox(seed))
        return (g.random(Ly * Lx) < p_up).astype(np.uint8)
    raise ValueError(f"unknown init {init!r}")


# ---------------------------------------------------------------------------
# The paper's window: T_max = log N / (lambda |dG_i|), N regions
# (PEs), |dG_i| the number of sites on a region's boundary, lambda the largest
# flip rate (reading #14/#15: natural log).  A bookkeeping formula for choosing
# W; it changes which windows the relaxation works on, never the trajectory.
# ---------------------------------------------------------------------------


def boundary_sites(bx: int, by: int) -> int:
    """|dG_i|: sites of a bx x by region with a neighbour outside it."""
    if bx == 1 or by == 1:
        return bx * by
    return 2 * bx + 2 * by - 4


def paper_tmax(n_regions: int, dG: int, lam: float = 1.0) -> float:
    return math.log(n_regions) / (lam * dG)


# ---------------------------------------------------------------------------
# BASELINE.json configs.  Readings #20/#21 fix what BASELINE.json leaves open.
# ---------------------------------------------------------------------------


@dataclasses.dataclass
class Workload:
    name: str
    Lx: int
    Ly: int
    bx: int
    by: int
    T: float
    J: float = 1.0
    H: float = 0.0
    init: str = "random"
    seed: int = 1
    W: float = 1.0
    t_end: float = 10.0
    rule: str = "metropolis"

    @property
    def n_regions(self) -> int:
        return (self.Lx // self.bx) * (self.Ly // self.by)

    @property
    def n_sites(self) -> int:
        return self.Lx * self.Ly

    def rates(self) -> List[float]:
        return rate_table(self.T, self.J, self.H, self.rule)

    def spins(self) -> np.ndarray:
        return initial_spins(self.Lx, self.Ly, self.init, self.seed)

    def n_windows(self) -> int:
        return int(math.ceil(self.t_end / self.W - 1e-12))

    def replace(self, **kw) -> "Workload":
        return dataclasses.replace(self, **kw)


CONFIGS = {
    # c1: 16x16, 4x4 regions, T=1.5, iid, W=1, t=10
    "c1": Workload("c1", 16, 16, 4, 4, T=1.5, W=1.0, t_end=10.0),
    # c2: 256x256, 8x8 regions, T=2.269, all up, W=0.375 (reading #20), t=100
    "c2": Workload("c2", 256, 256, 8, 8, T=2.269, init="up", W=0.375, t_end=100.0),
    # c3: 4096x4096, 16x16 regions, T=1, H=0.1, iid, W=2, t=200
    "c3": Workload("c3", 4096, 4096, 16, 16, T=1.0, H=0.1, W=2.0, t_end=200.0),
    # c4: 16384x16384, 4x4 regions, T=2, iid, W=0.5, t=50
    "c4": Workload("c4", 16384, 16384, 4, 4, T=2.0, W=0.5, t_end=50.0),
}


def c5_points() -> List[Workload]:
    """c5 sweep: 8192^2, b in {1,2,4,8,32} x T in {1,2.269,4} x W in {.25,1,4},
    t_end = 16 (reading #21)."""
    pts = []
    for b in (1, 2, 4, 8, 32):
        for T in (1.0, 2.269, 4.0):
            for W in (0.25, 1.0, 4.0):
                pts.append(Workload(f"c5_b{b}_T{T}_W{W}", 8192, 8192, b, b, T=T, W=W,
                                    t_end=16.0))
    return pts


def get(name: str, **overrides) -> Workload:
    w = CONFIGS[name]
    return w.replace(**overrides) if overrides else w


def exact_initial_rate_per_site(w: Workload, spins: Optional[np.ndarray] = None) -> float:
    """Sum_v r(class(v)) / L^2 at t=0 (bookkeeping for DESIGN.md tables).  Used
    only to size buffers and report; not part of either implementation."""
    s = w.spins() if spins is None else spins
    g = s.reshape(w.Ly, w.Lx).astype(np.int64)
    u = (np.roll(g, 1, 0) + np.roll(g, -1, 0) + np.roll(g, 1, 1) + np.roll(g, -1, 1))
    k = 5 * g + u
    r = np.array(w.rates())
    return float(r[k].mean())
