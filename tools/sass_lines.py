#!/usr/bin/env python
"""Join ncu per-SASS-instruction metrics with nvdisasm line info.

  python tools/sass_lines.py REPORT.ncu-rep LIB.so MANGLED_KERNEL [--launch I] [--depth outer|inner]

Aggregates "Warp Stall Sampling (All Samples)", "Instructions Executed" and
"Thread Instructions Executed" per source line: `outer` = the call site in the
kernel body (outermost 'inlined at' location), `inner` = the innermost line.
"""
import argparse
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def line_map(lib, kernel):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, check=True, capture_output=True)
    cub = [f for f in sorted(os.listdir(tmp)) if f.endswith(".cubin") and f.startswith("isr_runtime.")][0]
    out = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    inside = False
    cur = None
    pending = None
    m = {}
    for ln in out.splitlines():
        if ln.startswith("//--") and ".text." in ln:
            inside = ln.rstrip("- ").endswith(".text." + kernel)
            continue
        if not inside:
            continue
        if "//## File" in ln:
            locs = re.findall(r'"([^"]+)", line (\d+)', ln)
            loc = [(os.path.basename(f), int(n)) for f, n in locs]
            if pending is None or len(loc) >= len(pending):
                pending = loc  # several annotations may precede one instruction: keep the deepest
            continue
        mm = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if mm:
            if pending:
                cur = pending
            pending = None
            if cur:
                m[int(mm.group(1), 16)] = cur
    return m


def ncu_sections(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    secs = []
    for chunk in out.split('"Kernel Name"')[1:]:
        rows = list(csv.reader(io.StringIO('"Kernel Name"' + chunk)))
        hdr = rows[1]
        if secs and secs[-1][0] == rows[0][1] and secs[-1][2] == rows[2:]:
            continue  # ncu prints each launch's source table twice
        secs.append((rows[0][1], hdr, rows[2:]))
    return secs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("lib")
    ap.add_argument("kernel")
    ap.add_argument("--launch", type=int, default=0)
    ap.add_argument("--depth", default="outer")
    ap.add_argument("--top", type=int, default=40)
    args = ap.parse_args()
    lm = line_map(args.lib, args.kernel)
    secs = ncu_sections(args.report)
    name, hdr, rows = secs[args.launch]
    ia, iss, iie, ite = (hdr.index(c) for c in ("Address", "Warp Stall Sampling (All Samples)",
                                                "Instructions Executed", "Thread Instructions Executed"))
    base = int(rows[0][ia], 16)
    agg = collections.defaultdict(lambda: [0, 0, 0])
    tot = [0, 0, 0]
    for r in rows:
        off = int(r[ia], 16) - base
        locs = lm.get(off, [("?", 0)])
        if args.depth == "outer":
            key = locs[-1]
        elif args.depth == "inner":
            key = locs[0]
        else:  # integer: that many inlining levels below the outermost call site
            key = locs[max(-len(locs), -1 - int(args.depth))]
        v = [int(r[iss] or 0), int(r[iie] or 0), int(r[ite] or 0)]
        for i in range(3):
            agg[key][i] += v[i]
            tot[i] += v[i]
    print(f"{name}  launch {args.launch}: samples {tot[0]}  warp-inst {tot[1]:.3e}  thread-inst {tot[2]:.3e}")
    print(f"{'line':>28} {'stall%':>7} {'winst%':>7} {'tinst%':>7} {'thr/inst':>8}")
    for key, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[: args.top]:
        print(f"{key[0] + ':' + str(key[1]):>28} {100 * v[0] / max(tot[0], 1):7.2f} {100 * v[1] / max(tot[1], 1):7.2f} "
              f"{100 * v[2] / max(tot[2], 1):7.2f} {v[2] / max(v[1], 1):8.2f}")


if __name__ == "__main__":
    sys.exit(main())
