#!/usr/bin/env python
"""Per-CUDA-source-line instruction and stall attribution from an ncu report
(`--print-source cuda,sass`). Usage: python tools/ncu_lines.py rep.ncu-rep [--top 40]"""
import argparse
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--top", type=int, default=40)
a = ap.parse_args()
txt = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
fname, agg, hdr = "", [], None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or not r or r[0] == "" or r[0] == "Function Name":
        continue
    d = dict(zip(hdr[:2], r[:2]))
    num = lambda v: int(v) if v.strip().lstrip("-").isdigit() else 0
    ie = num(r[hdr.index("Instructions Executed")])
    st = num(r[hdr.index("Warp Stall Sampling (All Samples)")])
    agg.append((ie, st, f"{fname}:{r[0]}", r[1][:90]))
ti = sum(x[0] for x in agg) or 1
ts = sum(x[1] for x in agg) or 1
print(f"total warp instructions {ti}, stall samples {ts}")
for ie, st, loc, src in sorted(agg, key=lambda x: -x[1])[:a.top]:
    print(f"{100*ie/ti:5.1f}% inst {100*st/ts:5.1f}% stall  {loc:22s} {src}")
