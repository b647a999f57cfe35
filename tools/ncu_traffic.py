#!/usr/bin/env python
"""DRAM traffic of the K1 launches of one window (ncu --set full capture made
with tools/iter_profile.py --profile) against their algorithmic bytes.

  python tools/ncu_traffic.py REPORT.ncu-rep ITER_PROFILE_LOG OUT.json [--md OUT.md]

ITER_PROFILE_LOG holds iter_profile.py's JSON (per iteration: regions, ms,
algorithmic MB).  Writes per-launch and per-window totals; bench.py reads
OUT.json for roofline.traffic (DRAM bytes per launch of the dominant kernel).
"""
import csv
import io
import json
import subprocess
import sys


def main():
    rep, log, out = sys.argv[1:4]
    md = sys.argv[sys.argv.index("--md") + 1] if "--md" in sys.argv else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    iname, ird, iwr, idu = (h.index(k) for k in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                                  "gpu__time_duration.sum"))
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tscale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0}
    launches = []
    for r in rows[2:]:
        if "region_kernel" not in r[iname]:
            continue
        launches.append({"read": float(r[ird].replace(",", "")) * scale[units[ird]],
                         "write": float(r[iwr].replace(",", "")) * scale[units[iwr]],
                         "ms": float(r[idu].replace(",", "")) * tscale[units[idu]]})
    txt = open(log).read()
    prof = json.loads(txt[txt.index("["):txt.rindex("]") + 1])
    iters = prof[0]["iters"]
    n = min(len(iters), len(launches))
    # a recomputation moves S + 3H, H = 4 + 9 h (h = the
    # window's boundary-history entries per region)
    S, h = prof[0]["S"], prof[0]["h"] / prof[0]["nreg"]
    per_rec = S + 3 * (4 + 9 * h)
    alg = [iters[i]["regions"] * per_rec for i in range(n)]
    impl = [iters[i]["MB"] * 1e6 for i in range(n)]
    dram = [launches[i]["read"] + launches[i]["write"] for i in range(n)]
    res = {
        "kernel": rows[2][iname], "window": prof[0]["window"], "launches": n,
        "dram_bytes_per_launch": sum(dram) / n, "alg_bytes_per_launch": sum(alg) / n,
        "dram_over_alg": sum(dram) / sum(alg),
        "dram_over_impl": sum(dram) / sum(impl), "alg_bytes_per_recomputation": per_rec,
        "per_launch": [{"iteration": i + 1, "regions": iters[i]["regions"], "alg_bytes": alg[i],
                        "dram_read": launches[i]["read"], "dram_write": launches[i]["write"],
                        "ncu_ms": launches[i]["ms"]} for i in range(n)],
        "note": "ncu --set full --clock-control none: one capture of every K1 launch of one c4 window "
                "(cold caches, serialised); algorithmic bytes = SURVEY §8(d.3) A (S + 3H) with the window's "
                "measured h; dram_over_impl against the library's own count of touched bytes (DESIGN.md §6)",
    }
    json.dump(res, open(out, "w"), indent=1)
    if md:
        with open(md, "w") as f:
            f.write(f"# K1 DRAM traffic vs algorithmic bytes — c4 window {res['window']} ({n} launches)\n\n")
            f.write(f"kernel `{res['kernel']}`; {res['note']}\n\n")
            f.write("| it | regions | alg MB | DRAM read MB | DRAM write MB | DRAM/alg | ncu ms |\n|---|---|---|---|---|---|---|\n")
            for p in res["per_launch"]:
                d = p["dram_read"] + p["dram_write"]
                f.write(f"| {p['iteration']} | {p['regions']} | {p['alg_bytes'] / 1e6:.1f} | {p['dram_read'] / 1e6:.1f} | "
                        f"{p['dram_write'] / 1e6:.1f} | {d / max(p['alg_bytes'], 1):.2f} | {p['ncu_ms']:.3f} |\n")
            f.write(f"\nwindow: {res['alg_bytes_per_launch'] / 1e6:.1f} MB algorithmic and "
                    f"{res['dram_bytes_per_launch'] / 1e6:.1f} MB DRAM per launch (DRAM/alg = {res['dram_over_alg']:.2f})\n")
    print(json.dumps({k: v for k, v in res.items() if k != "per_launch"}))


if __name__ == "__main__":
    main()
