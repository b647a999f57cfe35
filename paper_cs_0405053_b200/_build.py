"""Build libising_sr.so in-tree for sm_100a (nvcc; no GPU needed to compile)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libising_sr.so")
SOURCES = [os.path.join(CSRC, f) for f in ("isr_runtime.cu", "isr_checkerboard.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("isr_region.cuh", "isr_warp.cuh", "isr_big.cuh", "isr_device.cuh", "isr_nccl.h",
                                                  "isr_peer.cuh")] + [
    os.path.join(os.path.dirname(PKG), "include", "ising_sr.h")]

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-fmad=false",          # no FMA contraction anywhere (bit parity)
    "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
    "-lineinfo",
    "-Xptxas", "-v",
    "-shared", "-Xcompiler", "-fPIC", "-ldl",
]


def nccl_include() -> list:
    """-I for NCCL >= 2.28's headers (nccl.h + the device API, nccl_device.h):
    the torch-bundled nvidia-nccl wheel.  Without them the library builds
    without the peer-memory exchange (isr_peer.cuh) and keeps send/recv."""
    import sysconfig
    for root in (sysconfig.get_paths().get("purelib"), "/opt/prime-rl/.venv/lib/python3.12/site-packages"):
        inc = os.path.join(root or "", "nvidia", "nccl", "include")
        if os.path.exists(os.path.join(inc, "nccl_device.h")):
            return ["-I", inc]
    return []


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS if os.path.exists(p))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [nvcc()] + NVCC_FLAGS + nccl_include() + ["-o", tmp] + SOURCES
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libising_sr.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, LIB)
    with open(os.path.join(PKG, "ptxas_report.txt"), "w") as f:
        f.write(res.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
