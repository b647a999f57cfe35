#!/usr/bin/env python
"""Registers / spills / smem per kernel from paper_cs_0405053_b200/ptxas_report.txt.
  python tools/regs.py [substring ...]"""
import os, re, sys
p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_cs_0405053_b200", "ptxas_report.txt")
cur = None
for ln in open(p):
    m = re.search(r"Compiling entry function '([^']+)'", ln)
    if m:
        cur = m.group(1)
        continue
    if cur and "spill" in ln:
        spill = ln.strip()
    if cur and "Used" in ln:
        if all(s in cur for s in sys.argv[1:]):
            print(f"{cur[:60]:60s} {ln.split(':',1)[1].strip()} | {spill}")
        cur = None
