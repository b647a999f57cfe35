"""P strips of one lattice as P library contexts on ONE device, driven
through the step-level C API with device-to-device copies as the transport.

This exercises exactly the multi-rank code path of the library (ghost rows,
pack/mark kernels, per-strip region ids and Philox keys, global flag
decision) without kernels that wait on one another: every iteration runs the
P strips one after the other and exchanges their ghost rows afterwards.  It is
the single-GPU stand-in for the NCCL strips of `dist.py` (shard invariance:
any P gives the same trajectory).
"""
from __future__ import annotations

from typing import List

import numpy as np
import torch

from .binding import IsingSR
from .dist import device_view


class LocalShards:
    def __init__(self, Lx, Ly, bx, by, rates, spins, W, t_end, seed, P: int, device: int = 0, **kw):
        self.P = P
        self.device = device
        self.sims: List[IsingSR] = [
            IsingSR(Lx, Ly, bx, by, rates, spins, W, t_end, seed, rank=q, world=P, device=device, **kw)
            for q in range(P)]
        self.g_hist: List[int] = []

    def _exchange(self):
        if self.P == 1:
            self.sims[0].exchange_done()
            return
        halos = [s.halo() for s in self.sims]
        dev = self.device
        for q, h in enumerate(halos):
            up, down = (q - 1) % self.P, (q + 1) % self.P
            for k in range(h.nchunks):
                n = h.chunk_bytes[k]
                device_view(halos[up].recv_from_down[k], n, dev).copy_(device_view(h.send_up[k], n, dev))
                device_view(halos[down].recv_from_up[k], n, dev).copy_(device_view(h.send_down[k], n, dev))
        torch.cuda.current_stream(dev).synchronize()
        for s in self.sims:
            s.exchange_done()

    def run_window(self, max_iterations: int = 1000) -> int:
        for s in self.sims:
            s.begin_window()
        it = 0
        while True:
            it += 1
            flags = [s.iterate() for s in self.sims]
            self._exchange()
            changed = max(f[0] for f in flags)
            overflow = max(f[1] for f in flags)
            if overflow:
                for s in self.sims:
                    s.end_iterations(-1)
                for s in self.sims:
                    s.begin_window()
                it = 0
                continue
            if not changed:
                for s in self.sims:
                    s.end_iterations(it)
                self.g_hist.append(it)
                return it
            if it >= max_iterations:
                raise RuntimeError("relaxation did not converge")

    def commit(self) -> int:
        return sum(s.commit() for s in self.sims)

    def spins(self) -> np.ndarray:
        return np.concatenate([s.spins() for s in self.sims])

    def digests(self):
        ds, cs = zip(*(s.digests() for s in self.sims))
        return np.concatenate(ds), np.concatenate(cs)

    def close(self):
        for s in self.sims:
            s.close()
