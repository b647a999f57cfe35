"""The multi-rank path through the public API on one GPU: 2 and 4 processes
(ranks) each own a strip, `run_window` calls the torch.distributed exchange
callback of `dist.py` every iteration (gloo with host staging here; NCCL on a
multi-GPU node), and the gathered result equals the oracle bit for bit.

No kernel waits on another rank's kernel: every exchange goes through the
host, so sharing one device between the ranks cannot deadlock."""
import os
import socket

import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, geom, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_cs_0405053_b200 import FLAG_DIGEST, IsingSR
        from paper_cs_0405053_b200.dist import make_exchange
        Lx, Ly, bx, by, T, W, t_end = geom
        w = workloads.Workload("dr", Lx, Ly, bx, by, T=T, W=W, t_end=t_end, seed=8)
        torch.cuda.set_device(0)
        ex = make_exchange(rank, world, 0, host_staging=True)
        sim = IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.spins(), w.W, w.t_end, w.seed, flags=FLAG_DIGEST,
                      rank=rank, world=world, device=0, exchange=ex)
        gs, ev = [], 0
        for _ in range(w.n_windows()):
            gs.append(sim.run_window())
            ev += sim.commit()
        dig, cnt = sim.digests()
        q.put((rank, ev, gs, sim.spins(), dig, cnt))
        sim.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("geom", [(32, 32, 4, 4, 2.269, 0.5, 3.0), (64, 64, 16, 16, 2.0, 1.0, 3.0)])
def test_ranks_through_run_window_bit_exact(world, geom):
    Lx, Ly, bx, by, T, W, t_end = geom
    if (Ly // by) % world:
        pytest.skip("strips must divide region rows")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, geom, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(world)), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
    w = workloads.Workload("dr", Lx, Ly, bx, by, T=T, W=W, t_end=t_end, seed=8)
    ref = oracle.des_workload(w)
    assert sum(r[1] for r in res) == ref["n_events"]
    assert all(r[2] == res[0][2] for r in res)  # every rank took the same global decisions
    assert np.array_equal(np.concatenate([r[3] for r in res]), ref["spins"])
    assert np.array_equal(np.concatenate([r[4] for r in res]), ref["digest"])
    assert np.array_equal(np.concatenate([r[5] for r in res]), ref["count"])
