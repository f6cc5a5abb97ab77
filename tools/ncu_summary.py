#!/usr/bin/env python
"""One-screen summary of an ncu --set full report: per launch the key counters and the top stall reasons
(python tools/ncu_summary.py report.ncu-rep > summary.txt)."""
import collections
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "launch__grid_size", "launch__registers_per_thread", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]


def main(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    ki = h.index("Kernel Name")
    for r in rows[2:]:
        print(r[ki][:110])
        for w in WANT:
            if w in h:
                i = h.index(w)
                print("    %-62s %16s %s" % (w, r[i], units[i]))
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                         text=True).stdout
    kern, hdr, data = None, None, collections.defaultdict(list)
    for r in csv.reader(src.splitlines()):
        if r and r[0] == "Kernel Name":
            kern = r[1]
            continue
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr and kern and len(r) == len(hdr):
            data[kern].append(r)
    for k, rs in data.items():
        cols = [i for i, x in enumerate(hdr) if x.startswith("stall_") and "(Not" not in x]
        tot = {hdr[i]: sum(float(r[i] or 0) for r in rs) for i in cols}
        s = sum(tot.values()) or 1.0
        top = sorted(((v / s, n[6:]) for n, v in tot.items() if v > 0), reverse=True)[:8]
        print("stalls %s: %s" % (k[:60], ", ".join("%s %.2f" % (n, v) for v, n in top)))


if __name__ == "__main__":
    main(sys.argv[1])
