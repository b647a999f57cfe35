"""Thin ctypes binding of libising_sr.so (include/ising_sr.h).

Argument marshalling only: every step of the simulation runs in the CUDA
kernels of the library.  There is no CPU fallback -- if the shared library
is missing this module raises at load time.
"""
from __future__ import annotations

import ctypes
import math
import os
from typing import Callable, Dict, Optional, Sequence, Tuple

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ISING_SR_LIB") or os.path.join(_PKG, "libising_sr.so")

FLAG_LOG_EVENTS = 0x1
FLAG_DIGEST = 0x2
FLAG_FRESH_WINDOW = 0x4  # alternate approach to subsequent steps
FLAG_OBSERVABLES = 0x8   # time integrals of M and of the bond sum per window
FLAG_JACOBI_ALL = 0x10   # recompute every region in every iteration (paper-faithful schedule)
FLAG_HALO_LOOPBACK = 0x20  # world == 1 + nccl_id: the wrap rows exchanged with itself over NCCL
FLAG_MAG_MOMENTS = 0x40   # time integrals of |M| and M^2 per window (device time sort of the log)

STATUS = {
    0: "OK", -1: "E_INVALID_ARG", -2: "E_DIMENSION", -3: "E_PARTITION", -4: "E_DIVERGED",
    -5: "E_CAPACITY", -6: "E_CUDA", -7: "E_NCCL", -8: "E_OOM", -9: "E_STATE",
}


class IsingSRError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {STATUS.get(status, status)}")


class Halo(ctypes.Structure):
    _fields_ = [("nchunks", ctypes.c_int32),
                ("send_up", ctypes.c_void_p * 4), ("send_down", ctypes.c_void_p * 4),
                ("recv_from_up", ctypes.c_void_p * 4), ("recv_from_down", ctypes.c_void_p * 4),
                ("chunk_bytes", ctypes.c_size_t * 4),
                ("flags", ctypes.c_void_p), ("stream", ctypes.c_void_p), ("row_bytes", ctypes.c_size_t)]


EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(Halo))
ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p)


class Config(ctypes.Structure):
    _fields_ = [("Lx", ctypes.c_int32), ("Ly", ctypes.c_int32),
                ("bx", ctypes.c_int32), ("by", ctypes.c_int32),
                ("J", ctypes.c_double), ("H", ctypes.c_double), ("T", ctypes.c_double),
                ("rate", ctypes.c_double * 10), ("W", ctypes.c_double), ("t_end", ctypes.c_double),
                ("seed", ctypes.c_uint64), ("max_iterations", ctypes.c_int32),
                ("hist_capacity", ctypes.c_int32), ("flags", ctypes.c_uint32),
                ("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("device", ctypes.c_int32),
                ("stream", ctypes.c_void_p), ("exchange", EXCHANGE_FN),
                ("exchange_user", ctypes.c_void_p),
                ("dev_alloc", ALLOC_FN), ("dev_free", FREE_FN), ("alloc_user", ctypes.c_void_p),
                ("nccl_id", ctypes.c_void_p), ("eq_quantum", ctypes.c_double), ("log_capacity", ctypes.c_int32)]


class Stats(ctypes.Structure):
    _fields_ = [("t_c", ctypes.c_double), ("windows", ctypes.c_int64),
                ("events_total", ctypes.c_int64), ("events_last_window", ctypes.c_int64),
                ("g_last", ctypes.c_int32), ("g_max", ctypes.c_int32),
                ("g_hist", ctypes.c_int64 * 64), ("f_last", ctypes.c_int32), ("f_max", ctypes.c_int32),
                ("iterations_total", ctypes.c_int64), ("overflow_retries", ctypes.c_int32),
                ("hist_capacity", ctypes.c_int32), ("recomputations_total", ctypes.c_int64),
                ("bytes_alg_last_window", ctypes.c_double), ("ms_last_window", ctypes.c_double),
                ("region_launches", ctypes.c_int64), ("region_ms", ctypes.c_double),
                ("region_bytes", ctypes.c_double),
                ("obs_M_last", ctypes.c_double), ("obs_B_last", ctypes.c_double),
                ("obs_M_total", ctypes.c_double), ("obs_B_total", ctypes.c_double),
                ("obs_time_total", ctypes.c_double),
                ("active_last", ctypes.c_int64 * 64),
                ("ms_exchange_total", ctypes.c_double), ("ms_commit_total", ctypes.c_double),
                ("obs_M_now", ctypes.c_int64), ("obs_B_now", ctypes.c_int64),
                ("edge_entries_last_window", ctypes.c_int64), ("log_replayed_last_window", ctypes.c_int64),
                ("ms_compact_total", ctypes.c_double),
                ("obs_absM_last", ctypes.c_double), ("obs_M2_last", ctypes.c_double),
                ("obs_absM_total", ctypes.c_double), ("obs_M2_total", ctypes.c_double)]


_lib = None

EXPORTS = ["ising_sr_init", "ising_sr_run_window", "ising_sr_commit", "ising_sr_run",
           "ising_sr_stats_get", "ising_sr_get_spins", "ising_sr_get_events", "ising_sr_get_digests",
           "ising_sr_begin_window", "ising_sr_iterate", "ising_sr_halo_get", "ising_sr_exchange_done",
           "ising_sr_end_iterations",
           "ising_sr_checkpoint_size", "ising_sr_checkpoint_save", "ising_sr_checkpoint_load",
           "ising_sr_launch_count", "ising_sr_destroy", "ising_sr_strerror", "ising_sr_nccl_unique_id",
           "ising_sr_struct_size",
           "ising_cb_sweeps", "ising_cb_run"]


def load_library(path: str = LIB_PATH):
    """Load libising_sr.so.  Raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} not found: build it with `python -m paper_cs_0405053_b200._build` "
                           "(or __graft_entry__.build()); there is no CPU fallback")
    L = ctypes.CDLL(path)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    L.ising_sr_init.argtypes = [ctypes.POINTER(Config), vp, ctypes.POINTER(vp)]
    L.ising_sr_run_window.argtypes = [vp, ctypes.POINTER(i32)]
    L.ising_sr_commit.argtypes = [vp, ctypes.POINTER(i64)]
    L.ising_sr_run.argtypes = [vp, ctypes.POINTER(i64)]
    L.ising_sr_stats_get.argtypes = [vp, ctypes.POINTER(Stats)]
    L.ising_sr_get_spins.argtypes = [vp, vp]
    L.ising_sr_get_events.argtypes = [vp, vp, vp, vp, i64, ctypes.POINTER(i64)]
    L.ising_sr_get_digests.argtypes = [vp, vp, vp]
    L.ising_sr_begin_window.argtypes = [vp]
    L.ising_sr_iterate.argtypes = [vp, vp]
    L.ising_sr_halo_get.argtypes = [vp, ctypes.POINTER(Halo)]
    L.ising_sr_exchange_done.argtypes = [vp]
    L.ising_sr_end_iterations.argtypes = [vp, i32]
    L.ising_sr_checkpoint_size.argtypes = [vp, ctypes.POINTER(i64)]
    L.ising_sr_checkpoint_save.argtypes = [vp, vp, i64]
    L.ising_sr_checkpoint_load.argtypes = [vp, vp, i64]
    L.ising_sr_launch_count.argtypes = [vp]
    L.ising_sr_launch_count.restype = i64
    L.ising_sr_destroy.argtypes = [vp]
    L.ising_sr_destroy.restype = None
    L.ising_sr_strerror.argtypes = [i32]
    L.ising_sr_strerror.restype = ctypes.c_char_p
    L.ising_sr_nccl_unique_id.argtypes = [vp]
    L.ising_sr_struct_size.argtypes = [i32]
    L.ising_sr_struct_size.restype = ctypes.c_size_t
    L.ising_cb_sweeps.argtypes = [vp, i32, i32, vp, ctypes.c_uint64, i64, i32, vp, vp]
    L.ising_cb_run.argtypes = [vp, vp, i32, i32, vp, ctypes.c_uint64, i64, i32, ctypes.POINTER(i64), i32]
    for name in EXPORTS:
        if name not in ("ising_sr_launch_count", "ising_sr_destroy", "ising_sr_strerror", "ising_sr_struct_size"):
            getattr(L, name).restype = i32
    _lib = L
    return L


def _check(status: int, where: str):
    if status != 0:
        raise IsingSRError(status, where)


def _current_stream_ptr(device: int) -> Optional[int]:
    """torch's current stream on `device`, or None (the library then creates
    its own stream) when that is the legacy default stream: its handle is 0,
    which the C ABI reads as "no stream"."""
    try:
        import torch
        if torch.cuda.is_available():
            h = torch.cuda.current_stream(device).cuda_stream
            return h or None
    except Exception:
        pass
    return None


def nccl_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (ising_sr_nccl_unique_id) for
    IsingSR(nccl_id=...): rank 0 creates it and broadcasts the bytes."""
    L = load_library()
    buf = ctypes.create_string_buffer(128)
    _check(L.ising_sr_nccl_unique_id(buf), "ising_sr_nccl_unique_id")
    return buf.raw


class IsingSR:
    """One shard (rank) of a synchronous-relaxation n-fold-way simulation.

    Mirrors the C ABI: ``run_window`` / ``commit`` / ``run`` / ``stats`` plus
    accessors.  ``spins`` is the full Ly*Lx lattice (1 = up)."""

    def __init__(self, Lx: int, Ly: int, bx: int, by: int, rates: Sequence[float], spins: Optional[np.ndarray],
                 W: float, t_end: float, seed: int = 1, *, J: float = 1.0, H: float = 0.0,
                 T: float = float("nan"), flags: int = FLAG_DIGEST, hist_capacity: int = 0,
                 max_iterations: int = 0, rank: int = 0, world: int = 1, device: int = 0,
                 stream: Optional[int] = None,
                 exchange: Optional[Callable[[Halo], int]] = None, torch_alloc: bool = False,
                 nccl_id: Optional[bytes] = None, eq_quantum: float = 0.0, log_capacity: int = 0):
        L = load_library()
        c = Config()
        c.Lx, c.Ly, c.bx, c.by = Lx, Ly, bx, by
        c.J, c.H, c.T = J, H, T
        for k in range(10):
            c.rate[k] = float(rates[k])
        c.W, c.t_end, c.seed = float(W), float(t_end), int(seed)
        c.max_iterations, c.hist_capacity, c.flags = max_iterations, hist_capacity, flags
        c.rank, c.world, c.device = rank, world, device
        c.stream = stream if stream else _current_stream_ptr(device)
        self._nccl_id = None
        if nccl_id is not None:
            if len(nccl_id) != 128:
                raise ValueError("nccl_id must be the 128 bytes of an ncclUniqueId")
            self._nccl_id = ctypes.create_string_buffer(bytes(nccl_id), 128)
            c.nccl_id = ctypes.cast(self._nccl_id, ctypes.c_void_p)
        c.eq_quantum = float(eq_quantum)
        c.log_capacity = int(log_capacity)
        self._cb = None
        if exchange is not None:
            def _tramp(user, halo_p):
                try:
                    return int(exchange(halo_p.contents))
                except Exception as e:  # pragma: no cover - surfaced as E_NCCL
                    import traceback
                    traceback.print_exc()
                    return 1
            self._cb = EXCHANGE_FN(_tramp)
            c.exchange = self._cb
        self._alloc_cbs = None
        if torch_alloc:  # device buffers from torch's caching allocator, on the ctx stream
            import torch
            st = c.stream

            def _alloc(nbytes, user):
                try:
                    return int(torch.cuda.caching_allocator_alloc(int(nbytes), device, st))
                except Exception:  # pragma: no cover - surfaced as E_OOM
                    return None

            def _free(ptr, user):
                torch.cuda.caching_allocator_delete(int(ptr))

            self._alloc_cbs = (ALLOC_FN(_alloc), FREE_FN(_free))
            c.dev_alloc, c.dev_free = self._alloc_cbs
        self.cfg = c
        self.Lx, self.Ly, self.bx, self.by, self.world, self.rank = Lx, Ly, bx, by, world, rank
        self.n_regions = (Lx // bx) * (Ly // by) // world
        sp = None  # spins None: the Philox init stream, generated on the device
        if spins is not None:
            s = np.ascontiguousarray(spins, dtype=np.uint8).reshape(-1)
            if s.shape[0] != Lx * Ly:
                raise ValueError("spins must hold Lx*Ly entries")
            sp = s.ctypes.data
        h = ctypes.c_void_p()
        _check(L.ising_sr_init(ctypes.byref(c), sp, ctypes.byref(h)), "ising_sr_init")
        self._h = h
        self._L = L

    # -- relaxation ---------------------------------------------------------
    def run_window(self) -> int:
        g = ctypes.c_int32()
        _check(self._L.ising_sr_run_window(self._h, ctypes.byref(g)), "ising_sr_run_window")
        return g.value

    def commit(self) -> int:
        ev = ctypes.c_int64()
        _check(self._L.ising_sr_commit(self._h, ctypes.byref(ev)), "ising_sr_commit")
        return ev.value

    def run(self) -> int:
        ev = ctypes.c_int64()
        _check(self._L.ising_sr_run(self._h, ctypes.byref(ev)), "ising_sr_run")
        return ev.value

    # step-level API (multi-rank drivers)
    def begin_window(self):
        _check(self._L.ising_sr_begin_window(self._h), "ising_sr_begin_window")

    def iterate(self) -> Tuple[int, int]:
        f = np.zeros(2, dtype=np.int32)
        _check(self._L.ising_sr_iterate(self._h, f.ctypes.data), "ising_sr_iterate")
        return int(f[0]), int(f[1])

    def halo(self) -> Halo:
        h = Halo()
        _check(self._L.ising_sr_halo_get(self._h, ctypes.byref(h)), "ising_sr_halo_get")
        return h

    def exchange_done(self):
        _check(self._L.ising_sr_exchange_done(self._h), "ising_sr_exchange_done")

    def end_iterations(self, g: int):
        _check(self._L.ising_sr_end_iterations(self._h, g), "ising_sr_end_iterations")

    # -- accessors ----------------------------------------------------------
    def stats(self) -> Dict[str, object]:
        s = Stats()
        _check(self._L.ising_sr_stats_get(self._h, ctypes.byref(s)), "ising_sr_stats_get")
        d = {name: getattr(s, name) for name, _ in Stats._fields_}
        d["g_hist"] = list(s.g_hist)
        d["active_last"] = list(s.active_last)
        return d

    def spins(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        """This rank's strip of committed spins, row-major uint8 (1 = up).
        `out`: optional caller buffer of that size (e.g. a pinned tensor's
        .numpy(), for a full-speed D2H copy)."""
        n = (self.Ly // self.world) * self.Lx
        if out is None:
            out = np.empty(n, dtype=np.uint8)
        elif out.dtype != np.uint8 or out.size != n or not out.flags["C_CONTIGUOUS"]:
            raise ValueError(f"out must be a contiguous uint8 array of {n} elements")
        _check(self._L.ising_sr_get_spins(self._h, out.ctypes.data), "ising_sr_get_spins")
        return out.reshape(-1)

    def events(self, cap: Optional[int] = None):
        n = ctypes.c_int64()
        _check(self._L.ising_sr_get_events(self._h, None, None, None, 0, ctypes.byref(n)), "ising_sr_get_events")
        m = n.value if cap is None else min(cap, n.value)
        t = np.zeros(max(m, 1), dtype=np.float64)
        r = np.zeros(max(m, 1), dtype=np.uint32)
        s = np.zeros(max(m, 1), dtype=np.uint16)
        _check(self._L.ising_sr_get_events(self._h, t.ctypes.data, r.ctypes.data, s.ctypes.data, m,
                                           ctypes.byref(n)), "ising_sr_get_events")
        return t[:m], r[:m], s[:m]

    def digests(self):
        d = np.zeros(self.n_regions, dtype=np.uint64)
        c = np.zeros(self.n_regions, dtype=np.uint64)
        want_d = bool(self.cfg.flags & FLAG_DIGEST)
        _check(self._L.ising_sr_get_digests(self._h, d.ctypes.data if want_d else None, c.ctypes.data),
               "ising_sr_get_digests")
        return (d if want_d else None), c

    def checkpoint(self) -> bytes:
        """The committed state at the current committed time (between windows)."""
        n = ctypes.c_int64()
        _check(self._L.ising_sr_checkpoint_size(self._h, ctypes.byref(n)), "ising_sr_checkpoint_size")
        buf = ctypes.create_string_buffer(n.value)
        _check(self._L.ising_sr_checkpoint_save(self._h, buf, n.value), "ising_sr_checkpoint_save")
        return buf.raw

    def restore(self, data: bytes):
        """Resume from checkpoint() of a ctx with the same configuration."""
        buf = ctypes.create_string_buffer(data, len(data))
        _check(self._L.ising_sr_checkpoint_load(self._h, buf, len(data)), "ising_sr_checkpoint_load")

    def launch_count(self) -> int:
        return int(self._L.ising_sr_launch_count(self._h))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._L.ising_sr_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def from_workload(w, *, spins: Optional[np.ndarray] = None, **kw) -> IsingSR:
    """Construct from a workloads.Workload-like object (fields Lx, Ly, bx, by,
    T, J, H, W, t_end, seed, rates(), spins())."""
    s = w.spins() if spins is None else spins
    return IsingSR(w.Lx, w.Ly, w.bx, w.by, w.rates(), s, w.W, w.t_end, w.seed,
                   J=w.J, H=w.H, T=w.T, **kw)


# ---------------------------------------------------------------------------
# second workload: checkerboard Metropolis sweeps (include/ising_sr.h, ising_cb_*)
# ---------------------------------------------------------------------------
def _probs(p: Sequence[float]) -> np.ndarray:
    a = np.ascontiguousarray(p, dtype=np.float64)
    if a.shape != (10,):
        raise ValueError("p must hold the 10 class probabilities")
    return a


def checkerboard_run(spins: np.ndarray, Lx: int, Ly: int, p: Sequence[float], seed: int, sweep0: int,
                     nsweeps: int, device: int = 0, out: Optional[np.ndarray] = None):
    """ising_cb_run: `nsweeps` checkerboard Metropolis sweeps of a host
    lattice (Ly*Lx uint8, 1 = up), starting at global sweep `sweep0`.
    Returns (spins, accepted flips)."""
    L = load_library()
    s = np.ascontiguousarray(spins, dtype=np.uint8).reshape(-1)
    if s.size != Lx * Ly:
        raise ValueError("spins must have Lx*Ly entries")
    if out is None:
        out = np.empty_like(s)
    elif out.dtype != np.uint8 or out.size != s.size or not out.flags["C_CONTIGUOUS"]:
        raise ValueError("out must be a contiguous uint8 array of Lx*Ly elements")
    pr = _probs(p)
    fl = ctypes.c_int64()
    _check(L.ising_cb_run(s.ctypes.data, out.ctypes.data, Lx, Ly, pr.ctypes.data, seed, sweep0, nsweeps,
                          ctypes.byref(fl), device), "ising_cb_run")
    return out.reshape(-1), int(fl.value)


def checkerboard_sweeps(d_spins: int, Lx: int, Ly: int, p: Sequence[float], seed: int, sweep0: int, nsweeps: int,
                        d_flips: Optional[int] = None, stream: Optional[int] = None, device: int = 0):
    """ising_cb_sweeps on a device-resident lattice (raw device pointers,
    e.g. tensor.data_ptr()); enqueued on `stream` (default: torch's current
    stream), not synchronised."""
    L = load_library()
    pr = _probs(p)
    st = stream if stream is not None else _current_stream_ptr(device)
    _check(L.ising_cb_sweeps(d_spins, Lx, Ly, pr.ctypes.data, seed, sweep0, nsweeps, d_flips, st),
           "ising_cb_sweeps")
