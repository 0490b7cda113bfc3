#!/usr/bin/env python
"""Summary of an ncu --set full capture exported on the GPU box as CSV
(`ncu -i rep --page raw --csv` and `--page source --csv --print-source sass`,
gzip): duration, issue / pipe utilisation, occupancy, DRAM bytes, top stall
reasons and the SASS lines with the most stall samples.
Usage: python tools/ncu_csv_summary.py RAW.csv [SASS.csv.gz] [--top 15]"""
import argparse
import csv
import gzip

ap = argparse.ArgumentParser()
ap.add_argument("raw")
ap.add_argument("sass", nargs="?")
ap.add_argument("--top", type=int, default=15)
a = ap.parse_args()
r = list(csv.reader(open(a.raw)))
h, u, v = r[0], r[1], r[2]
KEYS = [("gpu__time_duration.sum", "duration"), ("launch__registers_per_thread", "registers"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("sm__inst_executed.avg.per_cycle_active", "IPC"),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe cycles active %"),
        ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe instructions %"),
        ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe cycles active %"),
        ("lts__t_sector_hit_rate.pct", "L2 hit %"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"), ("smsp__inst_executed.sum", "warp instructions")]
print(f"kernel: {v[h.index('Kernel Name')][:100]}")
for k, name in KEYS:
    if k in h:
        print(f"  {name:28s} {v[h.index(k)]} {u[h.index(k)]}")
st = [(k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), float(v[h.index(k)] or 0))
      for k in h if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("_per_issue_active.ratio")]
print("  stall cycles per issued instruction: " + ", ".join(f"{n} {x:.2f}" for n, x in sorted(st, key=lambda t: -t[1])[:8]))
if a.sass:
    rr = list(csv.reader(gzip.open(a.sass, "rt")))
    hh = rr[1]
    rows = [x for x in rr[2:] if len(x) == len(hh)]
    num = lambda s: int(s) if s.strip().isdigit() else 0  # noqa: E731
    iS, iI, iSrc = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed"), hh.index("Source")
    ts = sum(num(x[iS]) for x in rows) or 1
    print(f"  top SASS lines by stall samples (of {ts}):")
    for k, x in sorted(enumerate(rows), key=lambda kx: -num(kx[1][iS]))[:a.top]:
        print(f"    #{k:5d} {100 * num(x[iS]) / ts:5.1f}%  exec {num(x[iI]):12d}  {x[iSrc].strip()[:70]}")
