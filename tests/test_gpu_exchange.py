"""The in-library strip exchange over NCCL, on one GPU.

FLAG_HALO_LOOPBACK makes a single strip read its wrap-around neighbours
through ghost rows that the library fills over a one-rank communicator --
the same code path, kernels and stream ordering as a multi-GPU strip run --
in both transports: ISING_SR_EXCHANGE=peer (the default: one fused kernel
stores the edge rows into the neighbours' ghost rows in an NCCL symmetric
window, exchanges the flags through an inbox and synchronises with the NCCL
device API's LSA barrier, isr_peer.cuh) and =sendrecv (ncclSend/ncclRecv to
itself and ncclAllReduce).  The
results must be the oracle's bit for bit; ISING_SR_K1_DELAY_NS makes K1
publish late, so an exchange that were not ordered after K1 on the library's
stream would move stale histories and break parity (or the g sequence).
"""
import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_cs_0405053_b200 import FLAG_DIGEST, FLAG_HALO_LOOPBACK, FLAG_LOG_EVENTS, nccl_unique_id  # noqa: E402
from _gpu_common import check_against_oracle, run_gpu  # noqa: E402


@pytest.mark.parametrize("exch", ["peer", "sendrecv"])
@pytest.mark.parametrize("env", [{}, {"ISING_SR_K1_DELAY_NS": "20000"}, {"ISING_SR_PIPELINE": "0"},
                                 {"ISING_SR_PIPELINE": "0", "ISING_SR_K1_DELAY_NS": "20000"}])
@pytest.mark.parametrize("geom", [
    # Lx, Ly, bx, by, T, W, t_end
    (32, 32, 4, 4, 2.269, 0.5, 3.0),
    (16, 24, 2, 2, 1.5, 1.0, 4.0),
    (32, 32, 8, 8, 2.0, 0.5, 3.0),
    (16, 16, 1, 1, 2.269, 0.5, 2.0),
    (64, 64, 16, 16, 2.269, 1.0, 3.0),
    (64, 32, 32, 32, 4.0, 0.5, 2.0),
    (32, 4, 4, 4, 2.0, 0.5, 3.0),      # one region row: the strip's first row is its last
])
def test_nccl_loopback_bit_exact(geom, env, exch, monkeypatch):
    monkeypatch.setenv("ISING_SR_EXCHANGE", exch)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    Lx, Ly, bx, by, T, W, t_end = geom
    w = workloads.Workload("loop", Lx, Ly, bx, by, T=T, W=W, t_end=t_end, seed=13)
    base = run_gpu(w)
    ref, gpu = check_against_oracle(w, flags=FLAG_DIGEST | FLAG_LOG_EVENTS | FLAG_HALO_LOOPBACK,
                                    nccl_id=nccl_unique_id())
    assert gpu["g"] == base["g"]  # the exchange adds no iterations
    st = gpu["stats"]
    assert st["ms_exchange_total"] > 0.0


@pytest.mark.parametrize("exch", ["peer", "sendrecv"])
def test_nccl_loopback_c4_prefix(exch, monkeypatch):
    """c4's full lattice (16384^2, 4x4 regions) through the NCCL loopback on
    the prefix t < 0.02: same digests, counts and spins as the oracle."""
    monkeypatch.setenv("ISING_SR_EXCHANGE", exch)
    import oracle
    w = workloads.get("c4", t_end=0.02)
    ref = oracle.des_workload(w)
    gpu = run_gpu(w, flags=FLAG_DIGEST | FLAG_HALO_LOOPBACK, nccl_id=nccl_unique_id())
    assert gpu["events"] == ref["n_events"]
    assert np.array_equal(gpu["count"], ref["count"])
    assert np.array_equal(gpu["digest"], ref["digest"])
    assert np.array_equal(gpu["spins"], ref["spins"])


@pytest.mark.parametrize("geom", [
    (32, 32, 4, 4, 2.269, 0.5, 3.0),
    (64, 64, 16, 16, 2.269, 1.0, 3.0),
])
def test_peer_exchange_in_graph_loop(geom, monkeypatch):
    """The fused peer-memory exchange has no host call, so strips can also run
    the device-side window loop (one CUDA graph per window with a conditional
    node, ISING_SR_GRAPH=1): bit-exact, with the same g as without strips."""
    monkeypatch.setenv("ISING_SR_EXCHANGE", "peer")
    monkeypatch.setenv("ISING_SR_GRAPH", "1")
    Lx, Ly, bx, by, T, W, t_end = geom
    w = workloads.Workload("loopg", Lx, Ly, bx, by, T=T, W=W, t_end=t_end, seed=17)
    base = run_gpu(w)
    ref, gpu = check_against_oracle(w, flags=FLAG_DIGEST | FLAG_LOG_EVENTS | FLAG_HALO_LOOPBACK,
                                    nccl_id=nccl_unique_id())
    assert gpu["g"] == base["g"]


def test_peer_exchange_capacity_growth(monkeypatch):
    """History capacity overflow with strips: every rank re-registers its
    symmetric window (collective) and restarts the window; still bit-exact."""
    monkeypatch.setenv("ISING_SR_EXCHANGE", "peer")
    w = workloads.Workload("loopcap", 32, 32, 4, 4, T=4.0, W=2.0, t_end=4.0, seed=19)
    ref, gpu = check_against_oracle(w, flags=FLAG_DIGEST | FLAG_LOG_EVENTS | FLAG_HALO_LOOPBACK,
                                    nccl_id=nccl_unique_id(), hist_capacity=1)
    assert gpu["stats"]["overflow_retries"] > 0
