"""CPU checks of the C-ABI boundary: the library builds, loads, exports every
entry point include/ising_sr.h declares, and validates its arguments before
touching a device."""
import ctypes
import os
import re

import numpy as np
import pytest

import workloads
from paper_cs_0405053_b200 import _build, binding

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return binding.load_library()


def _declared():
    src = open(os.path.join(ROOT, "include", "ising_sr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ising_sr_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for n in ("ising_sr_init", "ising_sr_run_window", "ising_sr_commit", "ising_sr_stats_get"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    for name in _declared():
        assert hasattr(lib, name), name
    # and the binding wraps all of them
    assert set(_declared()) <= set(binding.EXPORTS)


def test_no_oracle_symbols_in_product(lib):
    out = os.popen(f"nm -D {binding.LIB_PATH}").read()
    assert "orc_" not in out


def _cfg(**kw):
    w = workloads.get("c1")
    c = binding.Config()
    c.Lx, c.Ly, c.bx, c.by = kw.get("Lx", 16), kw.get("Ly", 16), kw.get("bx", 4), kw.get("by", 4)
    for k, r in enumerate(kw.get("rates", w.rates())):
        c.rate[k] = r
    c.W = kw.get("W", 1.0)
    c.t_end = kw.get("t_end", 10.0)
    c.world = kw.get("world", 1)
    c.rank = kw.get("rank", 0)
    c.flags = kw.get("flags", 0)
    c.eq_quantum = kw.get("eq_quantum", 0.0)
    return c


@pytest.mark.parametrize("kw,status", [
    (dict(Lx=2), -2), (dict(Ly=1), -2),
    (dict(bx=3), -3), (dict(Lx=18, bx=4), -3),
    (dict(W=float("nan")), -1), (dict(W=float("inf")), -1),   # W <= 0 selects the paper's T_max
    (dict(eq_quantum=-1.0), -1), (dict(eq_quantum=float("inf")), -1),
    (dict(flags=binding.FLAG_HALO_LOOPBACK), -1),              # loopback needs nccl_id
    (dict(rates=[-1.0] + [1.0] * 9), -1),
    (dict(bx=3, by=5, Lx=15, Ly=15), -1),        # unsupported region shape
    (dict(rank=3, world=2), -1),
])
def test_init_validation_errors(lib, kw, status):
    c = _cfg(**kw)
    spins = np.zeros(c.Lx * c.Ly, dtype=np.uint8)
    h = ctypes.c_void_p()
    assert lib.ising_sr_init(ctypes.byref(c), spins.ctypes.data, ctypes.byref(h)) == status
    assert not h.value


def test_null_arguments(lib):
    h = ctypes.c_void_p()
    assert lib.ising_sr_init(None, None, ctypes.byref(h)) == -1
    assert lib.ising_sr_run_window(None, None) == -1
    assert lib.ising_sr_commit(None, None) == -1
    lib.ising_sr_destroy(None)  # NULL-safe
    assert lib.ising_sr_launch_count(None) == 0


def test_strerror(lib):
    for s in range(0, -10, -1):
        msg = lib.ising_sr_strerror(s)
        assert msg and msg != b"unknown status"
    assert lib.ising_sr_strerror(-99) == b"unknown status"


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    monkeypatch.setattr(binding, "_lib", None)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        binding.load_library(str(tmp_path / "nope.so"))


def test_struct_layouts_match_the_library(lib):
    """The ctypes mirrors of ising_sr_config / ising_sr_stats / ising_sr_halo
    have the sizes the library was compiled with (a field added on one side
    only would shift every later field)."""
    assert lib.ising_sr_struct_size(0) == ctypes.sizeof(binding.Config)
    assert lib.ising_sr_struct_size(1) == ctypes.sizeof(binding.Stats)
    assert lib.ising_sr_struct_size(2) == ctypes.sizeof(binding.Halo)
    assert lib.ising_sr_struct_size(9) == 0
