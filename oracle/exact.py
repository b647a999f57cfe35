"""Exact equilibrium averages by enumeration -- TEST INFRASTRUCTURE.

The n-fold way with Metropolis or Glauber rates (eqs. pMin / pglauber,
P:166-181) satisfies detailed balance with respect to the Boltzmann weight
exp(-E/T) of eq. hamil, so long-time averages of its
continuous-time trajectory converge to the Boltzmann averages below.  This
is the plain definition: sum over all 2^(Lx*Ly) states.
"""
from __future__ import annotations

import numpy as np


def boltzmann_averages(Lx: int, Ly: int, T: float, J: float = 1.0, H: float = 0.0):
    """Return dict with <E>, <|M|>, <M^2>, <B>, <M> (M = sum s, B = sum over
    bonds counted once of s s', E = -J B - H M)."""
    n = Lx * Ly
    assert n <= 20
    idx = np.arange(2 ** n, dtype=np.int64)
    bits = ((idx[:, None] >> np.arange(n)) & 1).astype(np.int64)
    s = (2 * bits - 1).reshape(-1, Ly, Lx)
    M = s.sum(axis=(1, 2))
    B = (s * np.roll(s, -1, axis=1)).sum(axis=(1, 2)) + (s * np.roll(s, -1, axis=2)).sum(axis=(1, 2))
    E = -J * B - H * M
    w = np.exp(-(E - E.min()) / T)
    Z = w.sum()
    avg = lambda q: float((w * q).sum() / Z)
    return {"E": avg(E), "absM": avg(np.abs(M)), "M2": avg(M.astype(np.float64) ** 2),
            "B": avg(B), "M": avg(M)}
