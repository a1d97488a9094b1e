"""Summarise tools/prof_next.sh captures into profiles/<tag>_<op>_launches.csv and
profiles/<tag>_<op>_ncu_summary.md (launch list with each kernel's share of the step, and the key
metrics of the full capture: time, DRAM bytes vs the bench's algorithmic bytes, pipe activity).

usage: python tools/summarize_next.py gpurun_out/r01next r01"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

src_root, tag = sys.argv[1], sys.argv[2]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
prof = os.path.join(root, "profiles")

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
        "sm__cycles_elapsed.avg.per_second"]

for op in sorted(os.listdir(src_root)):
    d = os.path.join(src_root, op)
    if not os.path.exists(os.path.join(d, "prof.ncu-rep")):
        continue
    rows = [r for r in csv.reader(open(os.path.join(d, "launches.csv"))) if r and not r[0].startswith("==")]
    ix = {h: i for i, h in enumerate(rows[0])}
    launches = [(int(r[ix["ID"]]), r[ix["Kernel Name"]], float(r[ix["Metric Value"]])) for r in rows[1:]
                if r[ix["Metric Name"]] == "gpu__time_duration.sum"]
    with open(os.path.join(prof, f"{tag}_{op}_launches.csv"), "w") as f:
        f.write("id,kernel,gpu_time_ns\n")
        for i, k, t in launches:
            f.write(f'{i},"{k}",{t:.0f}\n')
    share = defaultdict(float)
    for _, k, t in launches:
        share[k.split("(")[0]] += t
    tot = sum(share.values())
    out = subprocess.run(["ncu", "-i", os.path.join(d, "prof.ncu-rep"), "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(out)))
    h, units = rr[0], rr[1]
    j = {x: i for i, x in enumerate(h)}
    caps = [{k: (r[j[k]], units[j[k]]) for k in KEYS if k in j} for r in rr[2:]]
    names = [r[j["Kernel Name"]] if "Kernel Name" in j else "?" for r in rr[2:]]
    try:
        bench = json.load(open(os.path.join(d, "bench.json")))
    except Exception:
        bench = {}
    lines = [f"# ncu summary {tag} / {op}", "",
             f"Command: `bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline` + the op's flags "
             f"(`tools/prof_next.sh`); launch list = `ncu --metrics gpu__time_duration.sum --clock-control none` "
             f"(cold-cache, serialised: use the SHARES, not the absolute times); full capture = "
             f"`ncu --set full --clock-control none --import-source on` of the op's main kernel.", ""]
    if bench:
        r = bench.get("roofline", {})
        lines += [f"bench (same box, not under ncu): value {bench.get('value'):.1f} {bench.get('unit')}, roofline "
                  f"{r.get('bound')} achieved {r.get('achieved'):.1f} {r.get('unit')} = {r.get('frac'):.3f} of {r.get('peak')}", ""]
    lines += ["## share of device time by kernel (launch list)", "", "| kernel | launches | share |", "|---|---|---|"]
    for k, t in sorted(share.items(), key=lambda x: -x[1]):
        n = sum(1 for _, kk, _ in launches if kk.split("(")[0] == k)
        lines.append(f"| `{k}` | {n} | {100 * t / tot:.1f}% |")
    lines += ["", "## full capture", "", "| metric | " + " | ".join(f"#{i}" for i in range(len(caps))) + " |",
              "|---|" + "---|" * len(caps), "| kernel | " + " | ".join(f"`{n[:60]}`" for n in names) + " |"]
    for k in KEYS:
        if caps and all(k in c for c in caps):
            lines.append(f"| {k} ({caps[0][k][1]}) | " + " | ".join(c[k][0] for c in caps) + " |")
    with open(os.path.join(prof, f"{tag}_{op}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print(op, "->", f"profiles/{tag}_{op}_ncu_summary.md", f"({len(launches)} launches, {len(caps)} captured)")
