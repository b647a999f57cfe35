#!/usr/bin/env python
"""Build compile-time variants of libising_sr.so into build_variants/<name>.so.

  python tools/build_variants.py name1=-DISR_X=1,-DISR_Y=0 name2=... [--jobs N]

Each variant is timed by pointing ISING_SR_LIB at it (bench.py, tests)."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_cs_0405053_b200 import _build  # noqa: E402


def one(spec):
    name, _, flags = spec.partition("=")
    out = os.path.join(ROOT, "build_variants", name + ".so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = ([_build.nvcc()] + _build.NVCC_FLAGS + _build.nccl_include() + [f for f in flags.split(",") if f] +
           ["-o", out] + _build.SOURCES)  # (the NCCL headers: without them a variant has no peer-memory exchange)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.stderr.write(r.stderr)
        raise SystemExit(f"variant {name} failed")
    regs = [ln for ln in r.stderr.splitlines() if "registers" in ln]
    return name, out


if __name__ == "__main__":
    specs = [a for a in sys.argv[1:] if not a.startswith("--")]
    with ThreadPoolExecutor(4) as ex:
        for name, out in ex.map(one, specs):
            print(name, out)
