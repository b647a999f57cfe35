"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic (no Philox event stream, no
exponential variates, no class logic, no event loop).  It only produces the
problem statement the paper starts from (§2):

* the lattice size, region size, J, H, T, window W and run length of each
  BASELINE.json config (c1..c5), and
* the initial spin configuration s(v), drawn iid from numpy's
  seeded generator, and
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
# "iid +-1 (p=0.5, seed s)" uses numpy's Philox bit generator (a documented,
# seeded generator; SURVEY reading #19 asks only for a fixed seeded stream).
# ---------------------------------------------------------------------------


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
        g = np.random.Generator(np.random.Philox(seed))
        if p_up == 0.5:
            # one random bit per site, drawn 64 at a time
            n = Ly * Lx
            words = g.integers(0, 2**63, size=(n + 62) // 63, dtype=np.int64)
            bits = ((words[:, None] >> np.arange(63, dtype=np.int64)) & 1).reshape(-1)[:n]
            return bits.astype(np.uint8)
        return (g.random(Ly * Lx) < p_up).astype(np.uint8)
    raise ValueError(f"unknown init {init!r}")


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
