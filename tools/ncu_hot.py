"""Summarise an ncu report: key raw metrics + per-instruction stall hot spots (source page)."""
import csv, io, subprocess, sys

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "launch__registers_per_thread", "sm__cycles_elapsed.avg.per_second",
            "lts__t_bytes.sum", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"]
    for w in want:
        if w in idx:
            print(f"{w:70s} {units[idx[w]]:8s} {[r[idx[w]] for r in rows[2:]]}")

def source(rep, kernel_idx=0, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows, hdr, k = [], None, -1
    for row in csv.reader(io.StringIO(out)):
        if row and row[0] == "Kernel Name":
            k += 1
            continue
        if row and row[0] == "Address":
            hdr = row
            continue
        if hdr and k == kernel_idx and len(row) > 5:
            rows.append(row)
    idx = {h: i for i, h in enumerate(hdr)}
    S, E = "Warp Stall Sampling (All Samples)", "Instructions Executed"
    tot = sum(int(r[idx[S]]) for r in rows)
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    print("samples", tot)
    # contiguous regions with the same execution count
    prev, acc, start, first = None, 0, None, ""
    regions = []
    for r in rows:
        e, s = int(r[idx[E]]), int(r[idx[S]])
        if e != prev:
            if prev is not None:
                regions.append((acc, start, last, prev, first))
            prev, acc, start, first = e, 0, r[0][-5:], r[1].strip()
        acc += s
        last = r[0][-5:]
    regions.append((acc, start, last, prev, first))
    for acc, a, b, e, f in sorted(regions, reverse=True)[:20]:
        print(f"region {a}-{b} exec={e:9d} samples={acc:6d} ({100*acc/tot:4.1f}%) first: {f[:60]}")
    print("top instructions:")
    for r in sorted(rows, key=lambda r: -int(r[idx[S]]))[:top]:
        s = int(r[idx[S]])
        st = sorted(((int(r[idx[h]]), h[6:]) for h in stalls), reverse=True)[:3]
        print(f"{s:6d} {100*s/tot:5.1f}% {r[0][-5:]} exec={int(r[idx[E]]):8d} {r[1].strip()[:58]:58s} {st}")

if __name__ == "__main__":
    rep = sys.argv[1]
    raw(rep)
    source(rep, int(sys.argv[2]) if len(sys.argv) > 2 else 0)
