#!/usr/bin/env python
"""Summarise an ncu report: headline metrics, stall reasons and the hottest
SASS basic blocks (by executed instructions).  Usage:
  python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--blocks 20] [--json out.json]
"""
import argparse
import csv
import io
import json
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"
KEYS = ["Duration", "Elapsed Cycles", "SM Active Cycles", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Grid Size", "Warp Cycles Per Issued Instruction",
        "Eligible Warps Per Scheduler", "Avg. Active Threads Per Warp", "Avg. Not Predicated Off Threads Per Warp",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Instructions"]


def run(args):
    return subprocess.run([NCU, "-i", *args], capture_output=True, text=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--blocks", type=int, default=20)
    ap.add_argument("--json")
    a = ap.parse_args()
    out = {"report": a.rep, "metrics": {}, "raw": {}}
    det = list(csv.reader(io.StringIO(run([a.rep, "--page", "details", "--csv"]))))
    if det:
        idx = {h: i for i, h in enumerate(det[0])}
        for row in det[1:]:
            name = row[idx["Metric Name"]]
            if name in KEYS:
                out["metrics"][name] = row[idx["Metric Value"]] + " " + row[idx["Metric Unit"]]
    raw = list(csv.reader(io.StringIO(run([a.rep, "--page", "raw", "--csv"]))))
    if len(raw) >= 3:
        hdr = raw[0]
        vals = raw[2]
        for h, v in zip(hdr, vals):
            if any(k in h for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fma_cycles_active",
                                    "sm__inst_executed_pipe_fma", "sm__pipe_alu_cycles_active",
                                    "smsp__average_warp_latency_issue_stalled", "smsp__pcsamp_warps_issue_stalled")):
                out["raw"][h] = v
    for k, v in out["metrics"].items():
        print(f"{k:45s} {v}")
    for k, v in sorted(out["raw"].items()):
        if "pcsamp" in k or "pipe" in k or "dram" in k:
            print(f"{k:75s} {v}")
    src = list(csv.reader(io.StringIO(run([a.rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    if len(src) > 2:
        hdr = src[1]
        ie, isr, ist = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
        data = [(int(r[ie] or 0), int(r[ist] or 0), r[isr].strip()) for r in src[2:] if len(r) > ie]
        tot = sum(d[0] for d in data) or 1
        tots = sum(d[1] for d in data) or 1
        blocks, cur = [], None
        for k, (ex, st, s) in enumerate(data):
            if cur and ex == cur[2]:
                cur[1] = k; cur[3] += st; cur[4] += 1
            else:
                if cur:
                    blocks.append(cur)
                cur = [k, k, ex, st, 1]
        blocks.append(cur)
        top = sorted(blocks, key=lambda b: -b[2] * b[4])[:a.blocks]
        print(f"\nhot SASS blocks (total warp instructions {tot:.3e}):")
        for b in sorted(top):
            print(f"  [{b[0]:5d}-{b[1]:5d}] n={b[4]:4d} x{b[2]:>11d} = {b[2] * b[4] / tot * 100:6.2f}% instr, "
                  f"{b[3] / tots * 100:6.2f}% stalls | {data[b[0]][2][:50]}")
        out["hot_blocks"] = [dict(start=b[0], end=b[1], n=b[4], exec=b[2], pct=b[2] * b[4] / tot * 100,
                                  stall_pct=b[3] / tots * 100, first=data[b[0]][2]) for b in sorted(top)]
    if a.json:
        json.dump(out, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    sys.exit(main())
