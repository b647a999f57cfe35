"""CPU oracle for the synchronous-relaxation n-fold way -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg (``cpu_baseline`` / ``--impl reference``) may import this package.  The
product package ``paper_cs_0405053_b200`` never imports it, and the two share
no code: the only common input is the ``workloads`` module (problem statement
and seeded initial spins, no method arithmetic).

The arithmetic lives in ``ising_oracle.c`` (plain C, gcc -O2
-ffp-contract=off); this module is ctypes marshalling plus two plain
definitions that need no C: the exact Boltzmann enumeration (``exact.py``).

Pins (tests/test_oracle_*.py): Philox known-answer vectors and an
independent implementation (ATen's philox_engine), E(U) against libm -log
within 4 ulp, closed-form dE / rate tables, the integer energy invariant
after every event, exact 3x3 Boltzmann averages, the T=inf closed form
m(t) = m0 exp(-2t), bit-exact reduction to the single-stream n-fold way when
one region covers the lattice, and a KS test against the single-stream
n-fold way.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Dict, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "ising_oracle.c")
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "ising_oracle.h"))):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call([
            "gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-Wall",
            "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


class _Cfg(ctypes.Structure):
    _fields_ = [("Lx", ctypes.c_int32), ("Ly", ctypes.c_int32),
                ("bx", ctypes.c_int32), ("by", ctypes.c_int32),
                ("rate", ctypes.c_double * 10), ("seed", ctypes.c_uint64),
                ("t_end", ctypes.c_double), ("t_obs0", ctypes.c_double),
                ("check", ctypes.c_int32), ("fresh_W", ctypes.c_double),
                ("eq_quantum", ctypes.c_double)]


class _Out(ctypes.Structure):
    _fields_ = [("digest", ctypes.c_void_p), ("count", ctypes.c_void_p),
                ("log_t", ctypes.c_void_p), ("log_region", ctypes.c_void_p),
                ("log_site", ctypes.c_void_p), ("log_cap", ctypes.c_int64),
                ("sample_t", ctypes.c_void_p), ("n_samples", ctypes.c_int32),
                ("sample_M", ctypes.c_void_p), ("sample_B", ctypes.c_void_p),
                ("n_events", ctypes.c_int64), ("log_n", ctypes.c_int64),
                ("obs", ctypes.c_double * 5), ("check_failures", ctypes.c_int32),
                ("n_bumps", ctypes.c_int64)]


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_philox4x32_10.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.orc_pair.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64,
                               ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
        L.orc_expvar.argtypes = [ctypes.c_double]
        L.orc_expvar.restype = ctypes.c_double
        L.orc_mix64.argtypes = [ctypes.c_uint64]
        L.orc_mix64.restype = ctypes.c_uint64
        L.orc_des_run.argtypes = [ctypes.POINTER(_Cfg), ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.POINTER(_Out)]
        L.orc_bkl_run.argtypes = [ctypes.POINTER(_Cfg), ctypes.c_uint32, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.POINTER(_Out)]
        L.orc_expvar_n.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
        L.orc_pair_n.argtypes = [ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
        L.orc_philox_n.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_int64]
        for name in ("orc_cand", "orc_breakpoint_budget"):
            getattr(L, name).restype = ctypes.c_double
        L.orc_cand.argtypes = [ctypes.c_double] * 3
        L.orc_breakpoint_budget.argtypes = [ctypes.c_double] * 4
        L.orc_fold.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        L.orc_fold.restype = ctypes.c_double
        L.orc_select.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                                 ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p]
        L.orc_class_counts.argtypes = [ctypes.c_int32] * 4 + [ctypes.c_void_p, ctypes.c_void_p]
        _lib = L
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


# -- scalar / batch primitives -------------------------------------------------

def philox(ctr: Sequence[int], key: Sequence[int]) -> tuple:
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_ptr(c), _ptr(k), _ptr(o))
    return tuple(int(x) for x in o)


def philox_n(ctr: np.ndarray, key: np.ndarray) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32).reshape(-1, 4)
    k = np.ascontiguousarray(key, dtype=np.uint32).reshape(-1, 2)
    o = np.zeros_like(c)
    lib().orc_philox_n(_ptr(c), _ptr(k), _ptr(o), c.shape[0])
    return o


def pair(seed: int, stream: int, n: int) -> tuple:
    U, V = ctypes.c_double(), ctypes.c_double()
    lib().orc_pair(seed, stream, n, ctypes.byref(U), ctypes.byref(V))
    return U.value, V.value


def pair_n(seed: int, stream: np.ndarray, idx: np.ndarray):
    s = np.ascontiguousarray(stream, dtype=np.uint32)
    i = np.ascontiguousarray(idx, dtype=np.uint64)
    U = np.zeros(s.shape[0], dtype=np.float64)
    V = np.zeros(s.shape[0], dtype=np.float64)
    lib().orc_pair_n(seed, _ptr(s), _ptr(i), _ptr(U), _ptr(V), s.shape[0])
    return U, V


def expvar(U: float) -> float:
    return lib().orc_expvar(U)


def expvar_n(U: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(U, dtype=np.float64)
    e = np.zeros_like(u)
    lib().orc_expvar_n(_ptr(u), _ptr(e), u.shape[0])
    return e


def mix64(z: int) -> int:
    return lib().orc_mix64(z)


def cand(t: float, R: float, lam: float) -> float:
    return lib().orc_cand(t, R, lam)


def breakpoint_budget(R: float, lam_old: float, t_b: float, t_s: float) -> float:
    return lib().orc_breakpoint_budget(R, lam_old, t_b, t_s)


def fold(N: Sequence[int], rates: Sequence[float]) -> float:
    n = np.ascontiguousarray(N, dtype=np.int32)
    r = np.ascontiguousarray(rates, dtype=np.float64)
    return lib().orc_fold(_ptr(n), _ptr(r))


def select(N: Sequence[int], rates: Sequence[float], V: float, lam: float):
    n = np.ascontiguousarray(N, dtype=np.int32)
    r = np.ascontiguousarray(rates, dtype=np.float64)
    k = np.zeros(1, dtype=np.int32)
    j = np.zeros(1, dtype=np.int64)
    lib().orc_select(_ptr(n), _ptr(r), V, lam, _ptr(k), _ptr(j))
    return int(k[0]), int(j[0])


def class_counts(Lx: int, Ly: int, bx: int, by: int, spins: np.ndarray) -> np.ndarray:
    s = np.ascontiguousarray(spins, dtype=np.uint8).reshape(-1)
    N = np.zeros(((Lx // bx) * (Ly // by), 10), dtype=np.int32)
    rc = lib().orc_class_counts(Lx, Ly, bx, by, _ptr(s), _ptr(N))
    if rc:
        raise ValueError(f"class_counts rc={rc}")
    return N


# -- whole-trajectory runs -----------------------------------------------------

def _cfg(Lx, Ly, bx, by, rates, seed, t_end, t_obs0=0.0, check=False, fresh_W=0.0, eq_quantum=0.0) -> _Cfg:
    c = _Cfg()
    c.Lx, c.Ly, c.bx, c.by = Lx, Ly, bx, by
    for k in range(10):
        c.rate[k] = float(rates[k])
    c.seed = seed
    c.t_end = float(t_end)
    c.t_obs0 = float(t_obs0)
    c.check = 1 if check else 0
    c.fresh_W = float(fresh_W)
    c.eq_quantum = float(eq_quantum)
    return c


def _run(kind: str, Lx: int, Ly: int, bx: int, by: int, rates: Sequence[float], seed: int,
         spins0: np.ndarray, t_end: float, *, log_cap: int = 0,
         sample_t: Optional[Sequence[float]] = None, t_obs0: float = 0.0,
         check: bool = False, stream: int = 0, fresh_W: float = 0.0,
         eq_quantum: float = 0.0) -> Dict[str, object]:
    nreg = 1 if kind == "bkl" else (Lx // bx) * (Ly // by)
    s0 = np.ascontiguousarray(spins0, dtype=np.uint8).reshape(-1)
    assert s0.shape[0] == Lx * Ly
    sout = np.zeros_like(s0)
    digest = np.zeros(nreg, dtype=np.uint64)
    count = np.zeros(nreg, dtype=np.uint64)
    lt = np.zeros(max(log_cap, 1), dtype=np.float64)
    lr = np.zeros(max(log_cap, 1), dtype=np.uint32)
    ls = np.zeros(max(log_cap, 1), dtype=np.uint16)
    st = None if sample_t is None else np.ascontiguousarray(sample_t, dtype=np.float64)
    ns = 0 if st is None else st.shape[0]
    sM = np.zeros(max(ns, 1), dtype=np.int64)
    sB = np.zeros(max(ns, 1), dtype=np.int64)
    o = _Out()
    o.digest, o.count = _ptr(digest), _ptr(count)
    o.log_t, o.log_region, o.log_site = _ptr(lt), _ptr(lr), _ptr(ls)
    o.log_cap = log_cap
    o.sample_t, o.n_samples = _ptr(st), ns
    o.sample_M, o.sample_B = _ptr(sM), _ptr(sB)
    cfg = _cfg(Lx, Ly, bx, by, rates, seed, t_end, t_obs0, check, fresh_W, eq_quantum)
    if kind == "bkl":
        rc = lib().orc_bkl_run(ctypes.byref(cfg), stream, _ptr(s0), _ptr(sout), ctypes.byref(o))
    else:
        rc = lib().orc_des_run(ctypes.byref(cfg), _ptr(s0), _ptr(sout), ctypes.byref(o))
    if rc != 0:
        raise ValueError(f"oracle {kind} run failed: rc={rc}")
    n = int(o.log_n)
    return {
        "spins": sout, "digest": digest, "count": count,
        "n_events": int(o.n_events),
        "log_t": lt[:n].copy(), "log_region": lr[:n].copy(), "log_site": ls[:n].copy(),
        "sample_M": sM[:ns].copy(), "sample_B": sB[:ns].copy(),
        "obs": list(o.obs), "check_failures": int(o.check_failures), "n_bumps": int(o.n_bumps),
    }


def des_run(Lx, Ly, bx, by, rates, seed, spins0, t_end, **kw):
    """O1: per-region-stream DES."""
    return _run("des", Lx, Ly, bx, by, rates, seed, spins0, t_end, **kw)


def bkl_run(Lx, Ly, rates, seed, spins0, t_end, stream: int = 0, **kw):
    """O2: single-stream textbook n-fold way over the whole lattice."""
    return _run("bkl", Lx, Ly, Lx, Ly, rates, seed, spins0, t_end, stream=stream, **kw)


def des_workload(w, t_end: Optional[float] = None, **kw):
    """Run O1 on a workloads.Workload."""
    return des_run(w.Lx, w.Ly, w.bx, w.by, w.rates(), w.seed, w.spins(),
                   w.t_end if t_end is None else t_end, **kw)


def cb_run(spins, Lx: int, Ly: int, p: Sequence[float], seed: int, sweep0: int, nsweeps: int):
    """Checkerboard Metropolis sweeps (orc_cb_run): returns (spins 0/1, flips)."""
    L = lib()
    L.orc_cb_run.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64,
                             ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]
    L.orc_cb_run.restype = ctypes.c_int
    s = np.ascontiguousarray(spins, dtype=np.uint8).reshape(-1).copy()
    if s.size != Lx * Ly:
        raise ValueError("spins must have Lx*Ly entries")
    pr = np.ascontiguousarray(p, dtype=np.float64)
    fl = ctypes.c_int64(0)
    rc = L.orc_cb_run(Lx, Ly, pr.ctypes.data, seed, sweep0, nsweeps, s.ctypes.data, ctypes.byref(fl))
    if rc != 0:
        raise ValueError("orc_cb_run: invalid arguments")
    return s, int(fl.value)
