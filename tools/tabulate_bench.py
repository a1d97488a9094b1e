"""One markdown row per bench JSON line in a directory (value, roofline fraction, per-M results, clocks).

usage: python tools/tabulate_bench.py gpurun_out/r01final2"""
import glob
import json
import os
import sys

src = sys.argv[1]
print("| file | workload / op / output | value | unit | roofline achieved / peak | frac | per M (Gpx/s, frac) | SM MHz |")
print("|---|---|---|---|---|---|---|---|")
for p in sorted(glob.glob(os.path.join(src, "bench_*.json"))):
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f"| {os.path.basename(p)} | unreadable: {e} | | | | | | |")
        continue
    c = d.get("config", {})
    r = d.get("roofline", {})
    per = d.get("per_M") or {}
    pm = ", ".join(f"{k}: {v.get('gpix_s', 0):.0f} / {v.get('frac_of_peak', 0):.3f}" for k, v in per.items())
    what = f"{c.get('workload')} / {c.get('op', 'encode')} / {c.get('output', 'f32')}" + (" / gop_phis" if c.get("gop_phis") else "")
    if d.get("impl") == "reference":
        what += " (reference arm)"
    ach = f"{r.get('achieved', 0):.0f} / {r.get('peak', 0):.0f} {r.get('unit', '')}" if r else ""
    frac = f"{r['frac']:.3f}" if r.get("frac") is not None else ""
    print(f"| {os.path.basename(p)} | {what} | {d.get('value', 0):.1f} | {d.get('unit')} | {ach} | {frac} | {pm} | "
          f"{(d.get('clocks') or {}).get('sm_mhz')} |")
