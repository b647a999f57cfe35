#!/usr/bin/env python
"""Markdown table of the first launches of an `ncu --page details --csv` dump.

  python tools/ncu_details_table.py DETAILS.csv TITLE [--n 6] > out.md
"""
import argparse
import csv

WANT = ['Duration', 'DRAM Throughput', 'Compute (SM) Throughput', 'Grid Size', 'Registers Per Thread',
        'Theoretical Occupancy', 'Achieved Occupancy', 'Issued Ipc Active', 'No Eligible',
        'Avg. Active Threads Per Warp', 'Branch Efficiency', 'L2 Hit Rate', 'Executed Instructions',
        'Warp Cycles Per Issued Instruction']


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("title")
    ap.add_argument("--n", type=int, default=6)
    args = ap.parse_args()
    rows = list(csv.reader(open(args.csv)))
    h = rows[0]
    i, nm, mv, mu, kn = (h.index(c) for c in ('ID', 'Metric Name', 'Metric Value', 'Metric Unit', 'Kernel Name'))
    d, names = {}, {}
    for r in rows[1:]:
        if r[nm] in WANT and int(r[i]) < args.n:
            d.setdefault(r[nm], {})[int(r[i])] = (r[mv] + ' ' + r[mu]).strip()
            names[int(r[i])] = r[kn].split('(')[0]
    print(f'## {args.title}\n')
    print('kernels: ' + ', '.join(f'it {j + 1}: `{names[j]}`' for j in sorted(names)) + '\n')
    print('| metric | ' + ' | '.join(f'it {j + 1}' for j in range(args.n)) + ' |')
    print('|---|' + '---|' * args.n)
    for k in WANT:
        print('| ' + k + ' | ' + ' | '.join(d.get(k, {}).get(j, '') for j in range(args.n)) + ' |')


if __name__ == '__main__':
    main()
