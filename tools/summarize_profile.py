"""Summarise a gpu_session run (launch list + ncu --set full capture) into profiles/<tag>_*.

usage: python tools/summarize_profile.py gpurun_out/r01c r01
Writes profiles/<tag>_launches.csv (kernel, duration), profiles/<tag>_ncu_summary.md and updates
profiles/ncu_traffic.json (per-launch DRAM bytes of the captured launches, read by bench.py)."""
import csv, io, json, os, subprocess, sys

src, tag = sys.argv[1], sys.argv[2]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
prof = os.path.join(root, "profiles")
os.makedirs(prof, exist_ok=True)

rows = [r for r in csv.reader(open(os.path.join(src, "launches.csv"))) if r and not r[0].startswith("==")]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
launches = [(int(r[ix["ID"]]), r[ix["Kernel Name"]], float(r[ix["Metric Value"]])) for r in rows[1:]
            if r[ix["Metric Name"]] == "gpu__time_duration.sum"]
with open(os.path.join(prof, f"{tag}_launches.csv"), "w") as f:
    f.write("id,kernel,gpu_time_ns\n")
    for i, k, t in launches:
        f.write(f'{i},"{k}",{t:.0f}\n')

out = subprocess.run(["ncu", "-i", os.path.join(src, "prof.ncu-rep"), "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(out)))
h, units = rr[0], rr[1]
j = {x: i for i, x in enumerate(h)}
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second",
        "lts__t_bytes.sum"]
cap = []
for r in rr[2:]:
    cap.append({k: (r[j[k]], units[j[k]]) for k in keys if k in j})

def mb(v, u):
    v = float(v)
    return v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(u, 1)

lines = [f"# ncu summary {tag}", "", f"source: `{src}` (gpu_session.sh): launch list = `ncu --metrics gpu__time_duration.sum "
         "--clock-control none` over `bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline` (cold-cache, serialised);",
         "full capture = `ncu --set full --clock-control none --import-source on -k regex:cs_measure -s 12 -c 4` (the four "
         "launches of the first timed step: M = 16, 32, 64, 128).", "",
         "## launch list (per-launch device time, ns)", "", "| id | kernel | time ns |", "|---|---|---|"]
for i, k, t in launches:
    lines.append(f"| {i} | `{k}` | {t:.0f} |")
tot = sum(t for _, _, t in launches)
lines += ["", f"All {len(launches)} launches are `cs_measure_kernel` (100% of device time in the step).", "",
          "## full capture (one launch per M)", "", "| metric | " + " | ".join(f"M={m}" for m in (16, 32, 64, 128)[:len(cap)]) + " |",
          "|---|" + "---|" * len(cap)]
for k in keys:
    if all(k in c for c in cap):
        lines.append(f"| {k} ({cap[0][k][1]}) | " + " | ".join(c[k][0] for c in cap) + " |")
traffic = {}
for m, c in zip((16, 32, 64, 128), cap):
    traffic[str(m)] = (mb(*c["dram__bytes_read.sum"]) + mb(*c["dram__bytes_write.sum"])) * 1e6
lines += ["", "DRAM traffic (read+write) per launch, bytes: " + json.dumps({k: round(v) for k, v in traffic.items()}),
          "(write bytes below the algorithmic output size mean the tail of the output was still in L2 when the kernel ended)"]
with open(os.path.join(prof, f"{tag}_ncu_summary.md"), "w") as f:
    f.write("\n".join(lines) + "\n")
tj = os.path.join(prof, "ncu_traffic.json")
d = json.load(open(tj)) if os.path.exists(tj) else {}
d["C4"] = {"per_M_bytes": traffic, "mean_bytes_per_launch": sum(traffic.values()) / len(traffic), "source": f"{tag}_ncu_summary.md"}
json.dump(d, open(tj, "w"), indent=1)
print("\n".join(lines))
