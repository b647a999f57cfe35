"""Shard invariance on one GPU: P strips (P library contexts with ghost rows,
pack/mark kernels and D2D exchange -- the multi-rank code path) give the
oracle's trajectory bit-exactly for every P."""
import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_cs_0405053_b200 import FLAG_DIGEST  # noqa: E402
from paper_cs_0405053_b200.local_shards import LocalShards  # noqa: E402


def _run(w, P, **kw):
    sh = LocalShards(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.spins(), w.W, w.t_end, w.seed, P, flags=FLAG_DIGEST, **kw)
    ev = 0
    nwin = w.n_windows()
    for _ in range(nwin):
        sh.run_window()
        ev += sh.commit()
    dig, cnt = sh.digests()
    out = {"events": ev, "spins": sh.spins(), "digest": dig, "count": cnt, "g": list(sh.g_hist)}
    sh.close()
    return out


@pytest.mark.parametrize("P", [1, 2, 4])
@pytest.mark.parametrize("geom", [(32, 32, 4, 4, 2.0, 0.5, 4.0), (16, 32, 2, 2, 2.269, 1.0, 4.0),
                                  (32, 16, 8, 4, 3.0, 0.7, 5.0)])
def test_strips_bit_exact(geom, P):
    Lx, Ly, bx, by, T, W, t_end = geom
    if (Ly // by) % P:
        pytest.skip("strips must divide region rows")
    w = workloads.Workload("sh", Lx, Ly, bx, by, T=T, W=W, t_end=t_end, seed=6)
    ref = oracle.des_workload(w)
    got = _run(w, P)
    assert got["events"] == ref["n_events"]
    assert np.array_equal(got["spins"], ref["spins"])
    assert np.array_equal(got["count"], ref["count"])
    assert np.array_equal(got["digest"], ref["digest"])


def test_strips_g_equals_single_strip_g():
    """Iterations per window do not depend on the strip count (the exchange
    happens every iteration; the fixed point is reached in the same g)."""
    w = workloads.Workload("gs", 32, 32, 4, 4, T=2.0, W=0.5, t_end=3.0, seed=9)
    a = _run(w, 1)
    b = _run(w, 4)
    assert a["g"] == b["g"]
    assert np.array_equal(a["digest"], b["digest"])


def test_strips_overflow_retry():
    w = workloads.Workload("so", 32, 32, 4, 4, T=4.0, W=2.0, t_end=4.0, seed=2)
    ref = oracle.des_workload(w)
    got = _run(w, 2, hist_capacity=1)
    assert np.array_equal(got["digest"], ref["digest"])
