#!/usr/bin/env python
"""Per-kernel HBM table from an `ncu --set full` capture of the HBM-bound
stages (tools/gpu_prof.sh: hbm_c4.ncu-rep, cfg4 Z-order): duration, DRAM
bytes (read + write), achieved GB/s and the fraction of the measured copy
bandwidth (MEASURED_PEAKS.json, else 6549.8 GB/s).
Usage: python tools/hbm_table.py rep.ncu-rep [--json out.json]"""
import argparse
import csv
import io
import json
import os
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--json")
ap.add_argument("--title", default="kernel (cfg4, 12.4M slots, Z-order)")
a = ap.parse_args()
peak = 6549.8
try:
    peak = float(json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"])
except (OSError, ValueError, KeyError):
    pass
txt = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv", "--metrics",
                      "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "usecond": 1e-6, "msecond": 1e-3}
out = []
print(f"{a.title:<44s} {'us':>7s} {'DRAM MB':>9s} {'GB/s':>8s} {'% of ' + str(round(peak)):>9s}")
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    f = lambda k: float(d[k].replace(",", "")) * scale.get(u[k], 1.0)  # noqa: E731
    t = f("gpu__time_duration.sum")
    by = f("dram__bytes_read.sum") + f("dram__bytes_write.sum")
    name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("crsh::", "")
    gbs = by / t / 1e9
    out.append({"kernel": name, "us": t * 1e6, "dram_bytes": by, "gbps": gbs, "frac": gbs / peak})
    print(f"{name:<44s} {t * 1e6:7.1f} {by / 1e6:9.1f} {gbs:8.1f} {100 * gbs / peak:9.1f}")
if a.json:
    json.dump({"peak_gbps": peak, "kernels": out}, open(a.json, "w"), indent=1)
