#!/usr/bin/env python
"""Per-kernel table from an ncu launch list (--metrics gpu__time_duration.sum
[,dram__bytes_read.sum,dram__bytes_write.sum] --csv --log-file X.csv).

Groups launches by kernel name over the frames of the timed region (the last
`--frames` occurrences of k_raygen or k_raygen_count start a frame) and prints mean duration,
share of the frame and DRAM bytes per launch.  ncu times are cold-cache and
serialised: compare shares, not absolutes (B200_PROFILING.md)."""
import argparse
import collections
import csv
import json
import re


def short(name):
    m = re.search(r"crsh::(\w+)", name)
    if m:
        return m.group(1)
    return name.split("(")[0][-40:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--frames", type=int, default=2)
    ap.add_argument("--json")
    a = ap.parse_args()
    rows = [r for r in csv.reader(open(a.csv)) if len(r) > 10]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    launches = collections.OrderedDict()
    for r in rows[1:]:
        lid = int(r[ix["ID"]])
        d = launches.setdefault(lid, {"name": short(r[ix["Kernel Name"]])})
        v = r[ix["Metric Value"]].replace(",", "")
        try:
            v = float(v)
        except ValueError:
            continue
        unit = r[ix["Metric Unit"]]
        name = r[ix["Metric Name"]]
        if name == "gpu__time_duration.sum":
            d["ns"] = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
        elif name.startswith("dram__bytes"):
            d[name] = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    ids = list(launches)
    starts = [i for i in ids if launches[i]["name"] in ("k_raygen", "k_raygen_count")]
    frames = starts[-a.frames:]
    agg = collections.OrderedDict()
    nf = 0
    for fi, s in enumerate(frames):
        end = frames[fi + 1] if fi + 1 < len(frames) else None
        sel = [i for i in ids if i >= s and (end is None or i < end) and launches[i]["name"].startswith("k_")]
        nf += 1
        for i in sel:
            d = launches[i]
            e = agg.setdefault(d["name"], {"n": 0, "ns": 0.0, "bytes": 0.0})
            e["n"] += 1
            e["ns"] += d.get("ns", 0.0)
            e["bytes"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot = sum(e["ns"] for e in agg.values()) or 1.0
    print(f"{'kernel':18s} {'launches/frame':>14s} {'us/frame':>10s} {'share':>7s} {'DRAM MB/launch':>15s}")
    out = {"frames": nf, "kernels": {}}
    for k, e in sorted(agg.items(), key=lambda kv: -kv[1]["ns"]):
        per = e["ns"] / nf / 1e3
        print(f"{k:18s} {e['n'] / nf:14.1f} {per:10.1f} {e['ns'] / tot * 100:6.1f}% {e['bytes'] / e['n'] / 1e6:15.3f}")
        out["kernels"][k] = {"launches_per_frame": e["n"] / nf, "us_per_frame": per, "share": e["ns"] / tot,
                             "dram_bytes_per_launch": e["bytes"] / e["n"]}
    print(f"{'total':18s} {'':14s} {tot / nf / 1e3:10.1f}")
    if a.json:
        json.dump(out, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
