"""World-size-2 (and 3) gloo tests of the strip-halo exchange protocol on CPU.

Checks that rank q's send_up lands in rank q-1's recv_from_down, its
send_down in rank q+1's recv_from_up (periodic), and that the flag
all-reduce is a MAX -- the host-side logic of the N>1 path."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_cs_0405053_b200.dist import halo_exchange, neighbours
        sizes = [5, 3 * 8, 3]
        su = [torch.full((n,), 10 * rank + 1, dtype=torch.uint8) for n in sizes]
        sd = [torch.full((n,), 10 * rank + 2, dtype=torch.uint8) for n in sizes]
        ru = [torch.zeros(n, dtype=torch.uint8) for n in sizes]
        rd = [torch.zeros(n, dtype=torch.uint8) for n in sizes]
        flags = torch.tensor([1 if rank == world - 1 else 0, 1 if rank == 0 else 0], dtype=torch.int32)
        halo_exchange(su, sd, ru, rd, flags, rank, world)
        up, down = neighbours(rank, world)
        ok = all(int(t[0]) == 10 * up + 2 and bool((t == t[0]).all()) for t in ru)
        ok &= all(int(t[0]) == 10 * down + 1 and bool((t == t[0]).all()) for t in rd)
        ok &= flags.tolist() == [1, 1]
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res[r] for r in range(world)), res


def test_strip_partition_rule():
    """Region rows split into equal contiguous strips; the C ABI rejects
    strips that do not divide (E_PARTITION)."""
    import ctypes
    import numpy as np
    from paper_cs_0405053_b200 import _build, binding
    _build.build()
    L = binding.load_library()
    c = binding.Config()
    c.Lx, c.Ly, c.bx, c.by = 16, 12, 4, 4   # 3 region rows
    for k in range(10):
        c.rate[k] = 1.0
    c.W, c.t_end, c.world, c.rank = 1.0, 1.0, 2, 0
    c.exchange = binding.EXCHANGE_FN(lambda u, h: 0)
    h = ctypes.c_void_p()
    s = np.zeros(16 * 12, dtype=np.uint8)
    assert L.ising_sr_init(ctypes.byref(c), s.ctypes.data, ctypes.byref(h)) == -3


def _id_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_cs_0405053_b200.dist import shared_nccl_id
        q.put((rank, shared_nccl_id(rank)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_shared_nccl_id_broadcast(world):
    """The bootstrap of the library's NCCL communicator (cfg.nccl_id): rank 0
    creates a 128-byte ncclUniqueId (ising_sr_nccl_unique_id, NCCL loaded by
    the library at run time) and every rank of the group receives the same
    bytes -- the only torch.distributed step of the N > 1 bench path."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_id_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    ids = [res[r] for r in range(world)]
    assert all(len(x) == 128 for x in ids) and all(x == ids[0] for x in ids) and any(ids[0])


# ---------------------------------------------------------------------------
# bench.py's N > 1 golden parity: the strips' spins and per-region counts
# hashed in rank order on rank 0 must equal the hashes of the whole lattice
# ---------------------------------------------------------------------------
class _FakeStrip:
    def __init__(self, spins, count, events):
        self._s, self._c, self._e = spins, count, events

    def digests(self):
        return None, self._c

    def spins(self):
        return self._s

    def stats(self):
        return {"events_total": self._e}


def _parity_worker(rank, world, port, q, path, corrupt):
    import numpy as np
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import types

        import bench
        rng = np.random.default_rng(5)
        Lx, Ly, b = 24, 12 * world, 4
        spins = rng.integers(0, 2, size=(Ly, Lx), dtype=np.uint8)
        count = rng.integers(0, 50, size=(Ly // b) * (Lx // b), dtype=np.uint32)
        rows, rr = Ly // world, (Ly // b) // world * (Lx // b)
        my_spins = spins[rank * rows:(rank + 1) * rows].copy()
        my_count = count[rank * rr:(rank + 1) * rr].copy()
        if corrupt and rank == world - 1:
            my_spins[0, 0] ^= 1
        sim = _FakeStrip(my_spins, my_count, int(my_count.sum()))
        w = types.SimpleNamespace(t_end=2.0, W=0.5)
        q.put((rank, bench.golden_parity("fake", sim, world, 4, w, rank, 0, path=path)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,corrupt", [(2, False), (3, False), (2, True)])
def test_bench_multi_rank_golden_parity(world, corrupt, tmp_path):
    import hashlib
    import json

    import numpy as np
    rng = np.random.default_rng(5)
    Lx, Ly, b = 24, 12 * world, 4
    spins = rng.integers(0, 2, size=(Ly, Lx), dtype=np.uint8)
    count = rng.integers(0, 50, size=(Ly // b) * (Lx // b), dtype=np.uint32)
    path = str(tmp_path / "g.json")
    json.dump({"t_end": 2.0, "n_events": int(count.sum()), "sha256_spins": hashlib.sha256(spins.tobytes()).hexdigest(),
               "sha256_count": hashlib.sha256(count.astype("<u8").tobytes()).hexdigest()}, open(path, "w"))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_parity_worker, args=(r, world, port, q, path, corrupt)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res[r] is None for r in range(1, world))
    assert res[0]["checked"] and res[0]["events"] and res[0]["counts"]
    assert res[0]["spins"] == (not corrupt) and res[0]["bit_exact"] == (not corrupt)
