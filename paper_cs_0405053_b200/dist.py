"""Multi-GPU strips: one process per GPU, torch.distributed plumbing.

The lattice's region rows are split into `world` contiguous strips (rank q
owns rows [q*RY/world, (q+1)*RY/world)).  After every relaxation iteration
each rank sends its first row's north-edge histories up and its last row's
south-edge histories down (periodic), receives the neighbours' into its ghost
rows, and all-reduces the {changed, overflow} flags with MAX -- the paper's
neighbour messages plus "synchronize".

Production path: the library does this itself over NCCL on its own stream
(`IsingSR(..., nccl_id=shared_nccl_id(rank))`): torch.distributed only
broadcasts the 128-byte ncclUniqueId once.  No Python runs per iteration.

`make_exchange` is the callback transport (include/ising_sr.h,
ising_sr_halo) kept for CPU-backend process groups: `halo_exchange` works on
torch tensors, so the same protocol runs over gloo with CPU tensors (the
world-size-2 CPU tests and the multi-process tests on one GPU).
"""
from __future__ import annotations

from typing import List, Sequence

import torch
import torch.distributed as dist


class _CudaView:
    """Minimal __cuda_array_interface__ exporter for a raw device pointer."""

    def __init__(self, ptr: int, nbytes: int, typestr: str = "|u1", itemsize: int = 1):
        self.__cuda_array_interface__ = {
            "shape": (nbytes // itemsize,), "typestr": typestr, "data": (int(ptr), False),
            "version": 3, "strides": None,
        }


def device_view(ptr: int, nbytes: int, device: int, typestr: str = "|u1", itemsize: int = 1) -> torch.Tensor:
    """Zero-copy torch view of library-owned device memory."""
    return torch.as_tensor(_CudaView(ptr, nbytes, typestr, itemsize), device=f"cuda:{device}")


def neighbours(rank: int, world: int):
    return (rank - 1) % world, (rank + 1) % world


def shared_nccl_id(rank: int, group=None) -> bytes:
    """The ncclUniqueId for the library's communicator: created by rank 0
    (ising_sr_nccl_unique_id), broadcast to every rank of `group`."""
    from .binding import nccl_unique_id
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def halo_exchange(send_up: Sequence[torch.Tensor], send_down: Sequence[torch.Tensor],
                  recv_from_up: Sequence[torch.Tensor], recv_from_down: Sequence[torch.Tensor],
                  flags: torch.Tensor, rank: int, world: int, group=None) -> None:
    """Strip-halo exchange + flag all-reduce (see module docstring).

    Message k going up carries tag 2k, going down tag 2k+1, so the pairing is
    unambiguous even when the up and down neighbour are the same rank
    (world == 2)."""
    up, down = neighbours(rank, world)
    ops: List[dist.P2POp] = []
    for k in range(len(send_up)):
        ops.append(dist.P2POp(dist.isend, send_up[k], up, group, 2 * k))
        ops.append(dist.P2POp(dist.irecv, recv_from_down[k], down, group, 2 * k))
        ops.append(dist.P2POp(dist.isend, send_down[k], down, group, 2 * k + 1))
        ops.append(dist.P2POp(dist.irecv, recv_from_up[k], up, group, 2 * k + 1))
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    dist.all_reduce(flags, op=dist.ReduceOp.MAX, group=group)


def make_exchange(rank: int, world: int, device: int, group=None, host_staging: bool = False):
    """Exchange callback for IsingSR(world > 1): wraps the library's device
    pointers (ising_sr_halo) as tensors and runs `halo_exchange` over NCCL.
    host_staging: copy through host memory (for a CPU backend such as gloo,
    e.g. several ranks on one device in tests)."""

    def _exchange(h) -> int:
        n = h.nchunks
        su = [device_view(h.send_up[k], h.chunk_bytes[k], device) for k in range(n)]
        sd = [device_view(h.send_down[k], h.chunk_bytes[k], device) for k in range(n)]
        ru = [device_view(h.recv_from_up[k], h.chunk_bytes[k], device) for k in range(n)]
        rd = [device_view(h.recv_from_down[k], h.chunk_bytes[k], device) for k in range(n)]
        fl = device_view(h.flags, 8, device, "<i4", 4)
        if not host_staging:
            # the collectives are ordered on the library's stream: they wait for
            # K1/pack and the library's next kernels wait for them
            with torch.cuda.stream(torch.cuda.ExternalStream(h.stream, device=device)):
                halo_exchange(su, sd, ru, rd, fl, rank, world, group)
            return 0
        torch.cuda.synchronize(device)
        hs = [[t.cpu() for t in ts] for ts in (su, sd)]
        hr = [[torch.empty_like(t, device="cpu") for t in ts] for ts in (ru, rd)]
        hf = fl.cpu()
        halo_exchange(hs[0], hs[1], hr[0], hr[1], hf, rank, world, group)
        for dst, src in zip(ru + rd + [fl], hr[0] + hr[1] + [hf]):
            dst.copy_(src)
        torch.cuda.synchronize(device)
        return 0

    return _exchange
