#!/usr/bin/env python
"""Markdown summary of an ncu --set full capture of K1 (first 6 launches + warp-state mix of launch 2).
  python tools/ncu_k1_md.py REPORT.ncu-rep TITLE > out.md"""
import csv, io, subprocess, sys

rep, title = sys.argv[1], sys.argv[2]
out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
i, nm, mv, mu = h.index('ID'), h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
want = ['Duration', 'DRAM Throughput', 'Compute (SM) Throughput', 'Grid Size', 'Registers Per Thread',
        'Theoretical Occupancy', 'Achieved Occupancy', 'Issued Ipc Active', 'No Eligible',
        'Avg. Active Threads Per Warp', 'Branch Efficiency', 'L2 Hit Rate', 'Executed Instructions']
d = {}
for r in rows[1:]:
    if r[nm] in want and int(r[i]) < 6:
        d.setdefault(r[nm], {})[int(r[i])] = (r[mv] + ' ' + r[mu]).strip()
print(f'# {title}\n')
print('Command: `ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:region_kernel '
      '-c 40 python tools/iter_profile.py --skip 20 --windows 1 --profile` (cold caches, serialised launches; '
      'durations are not bench numbers).\n')
print('| metric | it 1 | it 2 | it 3 | it 4 | it 5 | it 6 |\n|---|---|---|---|---|---|---|')
for k in want:
    print('| ' + k + ' | ' + ' | '.join(d.get(k, {}).get(j, '') for j in range(6)) + ' |')
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hh, vals = rr[0], rr[3]
outl = []
for hname, v in zip(hh, vals):
    if 'pcsamp_warps_issue_stalled' in hname and 'not_issued' not in hname:
        try:
            outl.append((float(v.replace(',', '')), hname.replace('smsp__pcsamp_warps_issue_stalled_', '')))
        except ValueError:
            pass
tot = sum(x for x, _ in outl)
print('\nWarp-state samples (share of all stall samples), iteration 2:\n\n| reason | share |\n|---|---|')
for x, n in sorted(outl, reverse=True)[:9]:
    print(f'| {n} | {100 * x / tot:.1f} % |')
