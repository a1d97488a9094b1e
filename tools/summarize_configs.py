"""Per-config DRAM traffic of K1 from one `ncu --set full` capture per workload (tools/diag_c3.sh):
-> profiles/<tag>_config_traffic.md and .json.  usage: python tools/summarize_configs.py DIR TAG"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402

WANT = {"gpu__time_duration.sum": "dur", "dram__bytes_read.sum": "dram_rd", "dram__bytes_write.sum": "dram_wr",
        "lts__t_sectors_srcunit_tex_op_read.sum": "l2_rd_sectors", "lts__t_sectors_srcunit_tex_op_write.sum": "l2_wr_sectors",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct"}
SCALE = {"us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for k, name in WANT.items():
        if k in hdr:
            i = hdr.index(k)
            v = float(vals[i].replace(",", ""))
            d[name] = v * SCALE.get(units[i], 1.0)
    return d


def main(src, tag):
    res = {}
    lines = [f"# K1 DRAM traffic per config ({tag}; `ncu --set full --clock-control none`, one launch each, "
             "`tools/run_one.py WL M` = planner plan, caches flushed by ncu before the replay)", "",
             "| config | M | µs (ncu) | DRAM read MB | alg. input MB | read / input | DRAM write MB | alg. output MB | L2 read MB | L2 read / DRAM read | tensor active | issue active |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for wl in ("C1", "C2", "C3", "C4", "C5"):
        rep = os.path.join(src, f"prof_{wl}.ncu-rep")
        if not os.path.exists(rep):
            continue
        cfg = synth.CONFIGS[wl]
        M = cfg.M
        nblk = -(-cfg.W // cfg.B) * -(-cfg.H // cfg.B)
        n_cs = cfg.S * (cfg.T - -(-cfg.T // cfg.G))
        alg_in = cfg.S * cfg.T * cfg.W * cfg.H
        alg_out = n_cs * nblk * M * 4
        d = raw(rep)
        l2 = d.get("l2_rd_sectors", 0) * 32
        row = {"M": M, "us": d["dur"] * 1e6, "dram_read": d["dram_rd"], "dram_write": d["dram_wr"], "alg_input": alg_in,
               "alg_output": alg_out, "l2_read": l2, "tensor_pct": d.get("tensor_pct"), "issue_pct": d.get("issue_pct")}
        res[wl] = row
        lines.append(f"| {wl} | {M} | {row['us']:.1f} | {d['dram_rd'] / 1e6:.1f} | {alg_in / 1e6:.1f} | {d['dram_rd'] / alg_in:.3f} | "
                     f"{d['dram_wr'] / 1e6:.1f} | {alg_out / 1e6:.1f} | {l2 / 1e6:.1f} | {l2 / max(d['dram_rd'], 1):.2f} | "
                     f"{d.get('tensor_pct', 0):.1f}% | {d.get('issue_pct', 0):.1f}% |")
    lines += ["", "DRAM write below the algorithmic output = the output tail still in L2 when the kernel ends "
              "(written back later, outside the launch). L2 read / DRAM read above 1 = strips or Φ slices re-read from L2 "
              "(key strips per unit, Φ K-slices per stage)."]
    with open(os.path.join(ROOT, "profiles", f"{tag}_config_traffic.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(os.path.join(ROOT, "profiles", f"{tag}_config_traffic.json"), "w") as f:
        json.dump(res, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
