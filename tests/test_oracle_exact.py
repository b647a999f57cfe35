"""Pins of oracle/exact.py (the Boltzmann enumeration the dynamics pins use)
against results derived independently of its code: the beta = 0 limit and
the hand-counted partition function of the 2x2 periodic lattice."""
import math

import numpy as np
import pytest

from oracle.exact import boltzmann_averages


@pytest.mark.parametrize("Lx,Ly", [(3, 3), (4, 3), (2, 5)])
def test_infinite_temperature_limit(Lx, Ly):
    """beta -> 0: independent fair spins, so <M> = 0, <B> = 0, <M^2> = N and
    <|M|> = sum_k |2k - N| C(N, k) / 2^N."""
    n = Lx * Ly
    a = boltzmann_averages(Lx, Ly, T=1e15, J=1.0, H=0.3)
    absm = sum(abs(2 * k - n) * math.comb(n, k) for k in range(n + 1)) / 2 ** n
    assert a["M"] == pytest.approx(0.0, abs=1e-9)
    assert a["B"] == pytest.approx(0.0, abs=1e-9)
    assert a["M2"] == pytest.approx(n, rel=1e-12)
    assert a["absM"] == pytest.approx(absm, rel=1e-12)


@pytest.mark.parametrize("T,J,H", [(1.0, 1.0, 0.0), (2.269, 1.0, 0.0), (1.7, 0.8, 0.25), (3.0, 1.0, -0.4)])
def test_two_by_two_partition_function(T, J, H):
    """2x2 periodic lattice, bonds counted once per site to the east and to
    the south (each physical pair twice): counting the 16 states by hand --
    all equal (M = +-4, B = 8), one flipped (M = +-2, B = 0; 4 states each),
    two adjacent flipped (M = 0, B = 0; 4 states), two diagonal flipped
    (M = 0, B = -8; 2 states)."""
    b = 1.0 / T
    classes = [(4, 8, 1), (-4, 8, 1), (2, 0, 4), (-2, 0, 4), (0, 0, 4), (0, -8, 2)]  # (M, B, multiplicity)
    w = [(m, bb, g * math.exp(b * (J * bb + H * m))) for m, bb, g in classes]
    Z = sum(x[2] for x in w)
    ref = {"M": sum(m * x for m, _, x in w) / Z, "B": sum(bb * x for _, bb, x in w) / Z,
           "M2": sum(m * m * x for m, _, x in w) / Z, "absM": sum(abs(m) * x for m, _, x in w) / Z}
    ref["E"] = -J * ref["B"] - H * ref["M"]
    a = boltzmann_averages(2, 2, T=T, J=J, H=H)
    for k in ("M", "B", "M2", "absM", "E"):
        assert a[k] == pytest.approx(ref[k], rel=1e-12, abs=1e-12), k
