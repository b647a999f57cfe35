#!/usr/bin/env python
"""Markdown table of a tools/sweep.py JSONL (c5 points or configs), with the
events/s of an earlier sweep beside it.

  python tools/sweep_md.py NEW.jsonl [--prev OLD.jsonl] [--title TEXT]
"""
import argparse
import json


def load(p):
    return {r["config"]: r for r in (json.loads(l) for l in open(p) if l.strip())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("new")
    ap.add_argument("--prev", default="")
    ap.add_argument("--title", default="")
    args = ap.parse_args()
    new = load(args.new)
    prev = load(args.prev) if args.prev else {}
    if args.title:
        print(args.title + "\n")
    hdr = "| point | b | T | W | g mean | g max | A | events/s |" + (" previous | ratio |" if prev else "") + " golden parity |"
    print(hdr)
    print("|" + "---|" * (hdr.count("|") - 1))
    n_ok = 0
    for name, r in new.items():
        ok = r.get("parity_golden")
        n_ok += ok is True
        row = (f"| {name} | {r['bx']} | {r['T']} | {r['W']:.4g} | {r['g_mean']:.1f} | {r['g_max']} | "
               f"{r['recomputations_per_region_window']:.1f} | {r['events_per_s']:.3e} |")
        if prev:
            p = prev.get(name)
            row += f" {p['events_per_s']:.3e} | {r['events_per_s'] / p['events_per_s']:.3f} |" if p else " | |"
        row += f" {'bit-exact' if ok else ('n/a' if ok is None else 'DIFFERS')} |"
        print(row)
    print(f"\n{n_ok}/{len(new)} points bit-exact against their golden")


if __name__ == "__main__":
    main()
