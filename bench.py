#!/usr/bin/env python
"""bench.py -- secondary Mrays/s of the CRSH path (BASELINE.json metric).

One step = one frame of the whole hot path through the C
ABI call crsh_trace_secondary: generate + hash + trim, compress, radix sort,
decompress, build, mesh cull, traversal, final tests, per-slot output (plus,
at N > 1, the library's own NCCL merge of the per-rank results, crsh_dist_init).

Default workload: BASELINE.json configs[3], the metric's configuration
("1920x1080 all secondary ray types, 1M triangles in 100 meshes"), seeded
synthetic scene + rasterised G-buffer (workloads/), with the R6 hash of
SURVEY §8(c) as `value` and the Z-order hash (NEXT-4) as `value_zorder`.
--config 2 selects configs[1] (the paper's 512x512 workload).  Timing: W
untimed warm-up frames, then K frames, each bracketed by CUDA events on the
launching stream after an L2 flush (a 512 MiB write outside the bracket);
barrier + synchronize on both sides; max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl crsh|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...    (hash-range sharding)
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "secondary Mrays/s at 1/2/4/8 B200; ray-primitive tests/ray vs naive N×M"
EQ9_FLOPS = 24      # Eq 9 test as evaluated: 3 sub, dot(5), 3 fma(6), dot(5), add, mul+fma(3), mul
MT_FLOPS = 46       # Moller-Trumbore as evaluated, reciprocal counted once
SM_COUNT, FP32_LANES, FMA_FLOPS = 148, 128, 2


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ----------------------------------------------------------------------------- clocks
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # the timed region starts once the sampler is live (nvidia-smi takes
            # ~0.5 s to start); samples from before it are dropped
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.02)
            self.lines.clear()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc and not self.lines:   # a region shorter than the 100 ms period: one reading right after it
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=10)
                self.lines.extend(ln.strip() for ln in out.stdout.splitlines() if ln.strip())
            except (OSError, subprocess.TimeoutExpired):
                pass
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 3:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
                bits = int(parts[2], 16)
            except ValueError:
                continue
            for b, name in REASONS.items():
                if bits & b and name != "gpu_idle":
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- helpers
def frame_flops(st):
    tests = int(np.asarray(st["tests"]).sum()) + int(sum(st["mesh_tests"]))
    return tests * EQ9_FLOPS + int(sum(st["final_tests"])) * MT_FLOPS


def eq9_evaluated(st):
    """Eq 9 tests k_traverse actually evaluated: the paper's counts of every
    level (and the object tree's cluster tests), minus the counted child tests
    the child prefilter proved failing without evaluating them, plus the
    prefilter's own tests (crsh_stats_t skipped_tests / prefilter_tests)."""
    return (int(np.asarray(st["tests"]).sum()) + int(sum(st.get("cluster_tests", [0])))
            - int(sum(st.get("skipped_tests", [0]))) + int(sum(st.get("prefilter_tests", [0]))))


def trav_flops(st):
    """FP32 work of k_traverse: the Eq 9 tests it evaluated and the
    Moller-Trumbore tests, from the frame's counters."""
    return eq9_evaluated(st) * EQ9_FLOPS + int(sum(st["final_tests"])) * MT_FLOPS


def load_traffic(config, zorder, world=1):
    """DRAM bytes (read + write) per launch of k_traverse from the committed
    ncu --set full capture of the same workload (profiles/r2_ncu/
    trav4_c4_{r6,z}_raw.csv: cfg4 on one GPU, the prefilter tree), with the
    capture's path; (None, None) for workloads without one."""
    if config != 4 or world != 1:
        return None, None
    rel = os.path.join("profiles", "r2_ncu", f"trav4_c4_{'z' if zorder else 'r6'}_raw.csv")
    try:
        import csv
        rows = list(csv.reader(open(os.path.join(ROOT, rel))))
        h, u, v = rows[0], rows[1], rows[2]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
        tot = sum(float(v[h.index(k)].replace(",", "")) * scale[u[h.index(k)]]
                  for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        return int(tot), rel
    except (OSError, ValueError, KeyError, IndexError):
        return None, None


def paper_context():
    """The paper's intersection-reduction figures with their hardware (context,
    not the target; BASELINE.json north_star): Table 4 totals as %
    of N x M and the reduction vs RAH, from the cited
    fixture tests/golden/paper_tables.json."""
    try:
        d = json.load(open(os.path.join(ROOT, "tests", "golden", "paper_tables.json")))
    except (OSError, ValueError):
        return None
    return {"hardware": "NVIDIA GeForce GTX TITAN 6 GB (Kepler GK110), CUDA + CUB (P:193-197)",
            "workload": "512x512, 2-level RSH, subdivision 8 (P:195)",
            "crsh_pct_of_brute": {t["scene"]: round(100.0 * t["CRSH"] / t["brute"], 2) for t in d["totals"]},
            "rah_pct_of_brute": {t["scene"]: round(100.0 * t["RAH"] / t["brute"], 2) for t in d["totals"]},
            "crsh_reduction_vs_rah_pct": {k: v for k, v in d["reduction_vs_rah_pct"].items() if k != "cite"},
            "cite": "Table 4 (P:259-265); P:231, P:253, P:303"}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


def oracle_band(w, flags, rows, prep=None):
    """Time the oracle (as it stands) on the centre band of `rows` image rows;
    returns (rays, seconds)."""
    import oracle
    from workloads.scenes import Workload
    prep = prep or oracle.ScenePrep(w.tris, w.mesh_ids)
    r0 = (w.height - rows) // 2
    P = w.width
    sub = Workload(w.name, w.tris, w.mesh_ids, w.tri_mat, w.materials, w.lights, w.eye, w.width, rows,
                   np.ascontiguousarray(w.pos.reshape(3, w.height, P)[:, r0:r0 + rows].reshape(3, -1)),
                   np.ascontiguousarray(w.nrm.reshape(3, w.height, P)[:, r0:r0 + rows].reshape(3, -1)),
                   np.ascontiguousarray(w.mat.reshape(w.height, P)[r0:r0 + rows].reshape(-1)), w.ray_types,
                   w.levels, w.leaf_size, w.branching)
    t0 = time.perf_counter()
    out = oracle.trace(sub, prep, flags=flags)
    return int(sum(out["stats"]["rays"])), time.perf_counter() - t0


def oracle_sample(w, flags, target_s=20.0):
    """Grow a centre band of image rows until one oracle run takes about
    target_s seconds of host CPU work (or the whole image); returns (rays,
    seconds, rows, cores)."""
    import oracle
    prep = oracle.ScenePrep(w.tris, w.mesh_ids)
    rows = 1
    while True:
        rays, dt = oracle_band(w, flags, rows, prep)
        if dt >= target_s / 2 or rows >= w.height:
            return rays, dt, rows, oracle.default_threads()
        rows = min(w.height, max(rows + 1, int(rows * min(8.0, target_s / max(dt, 1e-3)))))


# ----------------------------------------------------------------------------- GPU arm
def hbm_bytes(P, st, leaf_size):
    """Algorithmic HBM bytes of the hash/sort/build stages a1-a8 for one frame,
    SURVEY §8(d)'s per-ray model with c = chunks / rays:
    28 B per pixel of G-buffer read (28/rho per ray), then per ray 40 (ray
    record + key + value) + 4 + 8c (RLE) + 68c (4 onesweep passes of 8-bit
    digits) + 12c + 8 (decompression) + 4 + 32 + 32 (permutation, gather,
    sorted-ray write) + 64/B0 (nodes) = 120 + 88c + 64/B0."""
    n = int(sum(st["rays"]))
    c = int(sum(st["chunks"]))
    return 28 * P + n * (120 + 64.0 / leaf_size) + 88 * c


def _max_over_ranks(vals, world):
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def _barrier(world):
    import torch
    import torch.distributed as dist
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()


def measure(w, flags, args, local, world, flush, clocks=None):
    """W warm-up frames, then K frames each bracketed by CUDA events on the
    launching stream after an L2 flush (outside the bracket); barrier +
    synchronize on both sides; max over ranks. At N > 1 the scene is joined to
    the NCCL world (crsh_dist_init) and every frame includes the library's
    merge. Then 3 diagnostic frames with per-stage events (not timed)."""
    import torch

    import paper_2312_06538_b200 as crsh
    from paper_2312_06538_b200.api import tracer_for
    tr = tracer_for(w, device=local, flags=flags | crsh.F_KERNEL_TIMING)
    if args.dist_on:
        tr.dist_init()
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        tr.run(stream)
    merge_check = None
    if args.dist_on:   # the merged frame (every rank) equals this rank's own world-1 frame, bit for bit
        torch.cuda.synchronize()
        h, t = tr.hit_tri.clone(), tr.t.clone()
        ref = tracer_for(w, device=local, flags=flags)
        ref.run(stream)
        torch.cuda.synchronize()
        ok = torch.tensor([1 if (torch.equal(h, ref.hit_tri) and torch.equal(t.view(torch.int32), ref.t.view(torch.int32)))
                           else 0], dtype=torch.int32)
        import torch.distributed as dist
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        merge_check = "merged frame == world-1 frame on every rank" if int(ok) == 1 else "MISMATCH"
        del ref, h, t
    _barrier(world)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    trav = 0.0
    launches = 0
    import contextlib
    with (clocks if clocks is not None else contextlib.nullcontext()):
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            tr.run(stream)
            ev[i][1].record(stream)
            st = tr.stats()          # synchronises; outside the event bracket
            trav += st["stage_ms"][6]
            launches += tr.launches()
        torch.cuda.synchronize()
    _barrier(world)
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    st = tr.stats()
    merge = st["merge"]
    del tr
    # per-stage breakdown (diagnostic, outside the timed region): all stage events
    trs = tracer_for(w, device=local, flags=flags | crsh.F_STAGE_TIMING)
    if args.dist_on:
        trs.dist_init()
    stage = np.zeros(8)
    for k in range(4):
        flush.zero_()
        trs.run(stream)
        s_ = trs.stats()
        if k > 0:
            stage += np.asarray(s_["stage_ms"]) / 3
    del trs
    total_ms, trav_ms, *stage = _max_over_ranks([total_ms, trav / args.steps, *stage.tolist()], world)
    return dict(total_ms=total_ms, ms=total_ms / args.steps, trav_ms=trav_ms, stage=stage, st=st,
                launches=launches, merge=merge, merge_check=merge_check)


def config_dict(w, zorder, world, merge, objtree=False):
    return {"workload": w.name, "object_tree": bool(objtree), "pixels": w.width * w.height, "triangles": int(w.tris.shape[0]),
            "meshes": int(w.n_meshes), "ray_types": w.ray_types, "lights": int(w.lights.shape[0]),
            "levels": w.levels, "leaf_size": w.leaf_size, "branching": w.branching,
            "hash": "zorder" if zorder else "R6 (SPEC layout)",
            "parallelism": f"hash-range shard x{world}" if world > 1 else "single GPU", "merge": merge,
            "l2": "flushed before every timed step (512 MiB write outside the event bracket)"}


def run_crsh(args):
    import torch
    import torch.distributed as dist

    import paper_2312_06538_b200 as crsh
    from paper_2312_06538_b200.api import tracer_for
    from workloads import make_workload

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    args.dist_on = world > 1 or args.force_dist
    if world > 1:
        # host plumbing only (NCCL id broadcast, barriers, max over ranks): the
        # data path is libcrsh's own NCCL communicator (crsh_dist_init)
        dist.init_process_group("gloo")
    elif args.force_dist:   # the N > 1 code path with a world-1 NCCL communicator (tests)
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    base = crsh.F_SORT | crsh.F_MESH_CULL | (crsh.F_OBJTREE if args.objtree else 0)
    w = make_workload(args.config)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    clk = ClockSampler(local)
    main_z = bool(args.zorder)
    m = measure(w, base | (crsh.F_ZORDER if main_z else 0), args, local, world, flush, clk)
    other = None if args.single_hash else measure(w, base | (0 if main_z else crsh.F_ZORDER), args, local, world, flush)
    # NEXT-4 beside it: the Z-order hash with the object sphere-tree (reading O1)
    ztree = None if (args.single_hash or args.objtree) else measure(
        w, base | crsh.F_ZORDER | crsh.F_OBJTREE, args, local, world, flush)
    st = m["st"]
    rays = int(sum(st["rays"]))
    mrays = rays * args.steps / (m["total_ms"] * 1e-3) / 1e6
    # end to end through the public API with HOST buffers (crsh_trace_secondary_host):
    # G-buffer H2D from pinned memory and hit_tri / t D2H inside the timed region
    tr = tracer_for(w, device=local, flags=base | (crsh.F_ZORDER if main_z else 0))
    if args.dist_on:
        tr.dist_init()
    stream = torch.cuda.current_stream()
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    hpos, hnrm, hmat, hmats = pin(w.pos), pin(w.nrm), pin(w.mat), pin(w.materials)
    hh = torch.empty(tr.slots, dtype=torch.int32).pin_memory()
    ht = torch.empty(tr.slots, dtype=torch.float32).pin_memory()
    for _ in range(args.warmup):
        tr.run_host(hpos.numpy(), hnrm.numpy(), hmat.numpy(), hmats.numpy(), hh.numpy(), ht.numpy(), stream)
    _barrier(world)
    e_ms = 0.0
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        tr.run_host(hpos.numpy(), hnrm.numpy(), hmat.numpy(), hmats.numpy(), hh.numpy(), ht.numpy(), stream)
        b.record(stream)
        torch.cuda.synchronize()
        e_ms += a.elapsed_time(b)
    _barrier(world)
    e_ms = _max_over_ranks([e_ms], world)[0]
    P = w.width * w.height
    e2e = {"value": round(rays * args.steps / (e_ms * 1e-3) / 1e6, 3), "unit": "Mrays/s",
           "h2d_bytes_per_step": 28 * P + 12 * int(w.materials.shape[0]), "d2h_bytes_per_step": 8 * tr.slots,
           "api": "crsh_trace_secondary_host"}
    del tr
    if rank != 0:
        if args.dist_on:
            dist.destroy_process_group()
        return
    peaks = measured_peaks()
    clocks = clk.summary()
    sm_max = (clocks or {}).get("sm_max_mhz") or peaks.get("sm_max_mhz", 1965.0)
    peak_tflops, peak_src = SM_COUNT * FP32_LANES * FMA_FLOPS * sm_max * 1e6 / 1e12, "nominal 148 SM x 128 lanes x 2"
    try:   # measured FFMA throughput on this pool's B200 (tools/fp32_peak.cu)
        peak_tflops = float(json.load(open(os.path.join(ROOT, "profiles", "fp32_peak.json")))["ffma_tflops"])
        peak_src = "measured FFMA microbenchmark (profiles/fp32_peak.json)"
    except (OSError, ValueError, KeyError):
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6548.2))

    def kernel_roof(mm):
        s_ = mm["st"]
        fl = trav_flops(s_) / world          # per GPU: each rank traverses its share
        a_ = fl / (mm["trav_ms"] * 1e-3) / 1e12 if mm["trav_ms"] > 0 else 0.0
        fl_s = (eq9_evaluated(s_) * 28 + int(sum(s_["final_tests"])) * 55) / world
        a_s = fl_s / (mm["trav_ms"] * 1e-3) / 1e12 if mm["trav_ms"] > 0 else 0.0
        return a_, a_s

    def hbm_roof(mm):
        b_ = hbm_bytes(P, mm["st"], w.leaf_size)
        t_ = sum(mm["stage"][0:5])
        return b_, t_

    tfl, tfl_s = kernel_roof(m)
    hb, hms = hbm_roof(m)
    traffic, traffic_src = (None, None) if args.objtree else load_traffic(args.config, main_z, world)
    t_roof = hb / (hbm_peak * 1e9) * 1e3 + trav_flops(st) / world / (peak_tflops * 1e12) * 1e3
    tests_all, final_all = int(np.asarray(st["tests"]).sum()), int(sum(st["final_tests"]))
    brute = rays * w.tris.shape[0]
    out = {
        "metric": METRIC, "value": round(mrays, 3), "unit": "Mrays/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(m["ms"], 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded procedural scene + rasterised G-buffer, workloads/)",
        "config": config_dict(w, main_z, world, crsh.MERGE.get(m["merge"], str(m["merge"])), args.objtree),
        "rays_per_step": rays,
        "tests_per_ray": round((tests_all + final_all) / max(rays, 1), 2),
        "tests_by_level": {f"L{k}": int(np.asarray(st["tests"])[:, k].sum()) for k in range(w.levels, 0, -1)},
        "hits_by_level": {f"L{k}": int(np.asarray(st["hits"])[:, k].sum()) for k in range(w.levels, 0, -1)},
        "final_tests": final_all, "mesh_tests": int(sum(st["mesh_tests"])),
        "naive_tests_per_ray": int(w.tris.shape[0]),
        "relative_pct_of_brute": round(100.0 * (tests_all + final_all) / max(brute, 1), 4),
        "stage_ms": {n: round(v, 4) for n, v in zip(crsh.STAGES, m["stage"])},
        "roofline": {
            "bound": "alu", "kernel": "k_traverse (a9-a12, the dominant kernel)", "achieved": round(tfl, 3),
            "peak": round(peak_tflops, 2), "unit": "TFLOP/s", "frac": round(tfl / peak_tflops, 4), "traffic": traffic,
            "flops_convention": f"{EQ9_FLOPS} flops per Eq 9 test and {MT_FLOPS} per Moller-Trumbore test, the "
                                f"operations of the evaluated formulas (DESIGN.md §5); with SURVEY §8(d)'s estimates "
                                f"(28 / 55) frac = {tfl_s / peak_tflops:.4f}; Eq 9 tests counted as evaluated: the "
                                f"paper's counts - tests skipped by the prefilter "
                                f"({int(sum(st.get('skipped_tests', [0])))}) + prefilter tests "
                                f"({int(sum(st.get('prefilter_tests', [0])))})",
            "frac_survey_convention": round(tfl_s / peak_tflops, 4),
            "note": f"peak: {peak_src}; kernel time from CUDA events around k_traverse on the frame's stream, "
                    f"per GPU; traffic: DRAM read + write bytes per launch from "
                    f"{traffic_src or 'no committed capture of this workload (null)'}",
            "hbm_stages": {"bound": "hbm", "stages": "a1-a8 (generate+trim, compress, sort, decompress, build)",
                           "bytes": int(hb), "ms": round(hms, 4), "achieved": round(hb / (hms * 1e-3) / 1e9, 1),
                           "peak": hbm_peak, "unit": "GB/s", "frac": round(hb / (hms * 1e-3) / 1e9 / hbm_peak, 4),
                           "bytes_model": "SURVEY §8(d): 28 B/pixel + (120 + 88 c + 64/B0) B/ray, c = chunks/rays"},
            "end_to_end": {"t_roof_ms": round(t_roof, 4), "t_measured_ms": round(m["ms"], 4),
                           "frac": round(t_roof / m["ms"], 4),
                           "model": "t_roof = a1-a8 bytes / HBM peak + traversal flops per GPU / FP32 peak"},
        },
        "gpu_launches": m["launches"],
        "merge_check": m["merge_check"],
        "e2e": e2e,
        "paper_context": paper_context(),
        "clocks": clocks,
    }
    if other is not None:
        so = other["st"]
        ro = int(sum(so["rays"]))
        to = int(np.asarray(so["tests"]).sum()) + int(sum(so["final_tests"]))
        oa, _ = kernel_roof(other)
        ob, oms = hbm_roof(other)
        key = "r6" if main_z else "zorder"
        out[f"value_{key}"] = round(ro * args.steps / (other["total_ms"] * 1e-3) / 1e6, 3)
        out[f"ms_per_step_{key}"] = round(other["ms"], 4)
        out[f"tests_per_ray_{key}"] = round(to / max(ro, 1), 2)
        out[f"relative_pct_of_brute_{key}"] = round(100.0 * to / max(ro * w.tris.shape[0], 1), 4)
        out[f"roofline_{key}"] = {"k_traverse_frac": round(oa / peak_tflops, 4),
                                  "hbm_stages_frac": round(ob / (oms * 1e-3) / 1e9 / hbm_peak, 4),
                                  "hbm_stages_ms": round(oms, 4),
                                  "stage_ms": {n: round(v, 4) for n, v in zip(crsh.STAGES, other["stage"])}}
        out["gpu_launches"] += other["launches"]
    if ztree is not None:
        sz = ztree["st"]
        rz = int(sum(sz["rays"]))
        tz = int(np.asarray(sz["tests"]).sum()) + int(sum(sz["final_tests"]))
        za, _ = kernel_roof(ztree)
        out["value_zorder_objtree"] = round(rz * args.steps / (ztree["total_ms"] * 1e-3) / 1e6, 3)
        out["ms_per_step_zorder_objtree"] = round(ztree["ms"], 4)
        out["tests_per_ray_zorder_objtree"] = round(tz / max(rz, 1), 2)
        out["cluster_tests_zorder_objtree"] = int(sum(sz["cluster_tests"]))
        out["roofline_zorder_objtree"] = {"k_traverse_frac": round(za / peak_tflops, 4),
                                          "stage_ms": {n: round(v, 4) for n, v in zip(crsh.STAGES, ztree["stage"])}}
        out["gpu_launches"] += ztree["launches"]
    if world == 1 and not args.no_cpu_baseline:
        cr, cs, rows, cores = oracle_sample(w, base | (crsh.F_ZORDER if main_z else 0))
        out["cpu_baseline"] = {"value": round(cr / cs / 1e6, 5), "unit": "Mrays/s", "cores": cores, "kind": "oracle",
                               "sample": f"{rows} of {w.height} image rows (centre band), {cr} rays, {cs:.1f} s"}
    print(json.dumps(out), flush=True)
    if args.dist_on:
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- reference arm (the oracle)
def run_reference(args):
    rank, world, local = env_rank()
    if rank != 0:
        return
    import oracle
    from workloads import make_workload
    oracle.build()
    w = make_workload(args.config)
    flags = 3 | (4 if args.zorder else 0) | (64 if args.objtree else 0)
    budget = 150.0 / max(1, args.steps + args.warmup)      # whole run within a few minutes
    rows_probe = oracle_sample(w, flags, target_s=min(budget, 8.0))[2]
    prep = oracle.ScenePrep(w.tris, w.mesh_ids)
    times, rays = [], 0
    for i in range(args.warmup + args.steps):
        r, dt = oracle_band(w, flags, rows_probe, prep)
        if i >= args.warmup:
            times.append(dt)
            rays += r
    v = rays / sum(times) / 1e6
    out = {"metric": METRIC, "value": round(v, 5), "unit": "Mrays/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(1e3 * sum(times) / len(times), 2), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
           "config": config_dict(w, bool(args.zorder), 1, "none", args.objtree),
           "cpu_baseline": {"value": round(v, 5), "unit": "Mrays/s", "cores": oracle.default_threads(),
                            "kind": "oracle", "sample": f"{rows_probe} of {w.height} image rows per step"},
           "e2e": {"value": round(v, 5), "unit": "Mrays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ----------------------------------------------------------------------------- extra reports (not the contract line)
def _time_frames(tr, steps, stream):
    import torch
    ms = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        tr.run(stream)
        b.record(stream)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return float(np.median(ms))


def run_table4(args):
    """The paper's Table 4 comparison on the synthetic workload:
    total ray-primitive tests and frame time of CRSH, CRSH with the Z-order
    hash, RAH (no sort, no mesh culling) and naive N x M."""
    import torch

    import paper_2312_06538_b200 as crsh
    from paper_2312_06538_b200.api import tracer_for
    from workloads import make_workload
    w = make_workload(args.config)
    stream = torch.cuda.current_stream()
    rows = {}
    for name, flags in (("brute", crsh.F_BRUTE), ("rah", 0), ("crsh", 3), ("crsh_zorder", 7),
                        ("crsh_objtree", 3 | crsh.F_OBJTREE), ("crsh_zorder_objtree", 7 | crsh.F_OBJTREE)):
        tr = tracer_for(w, flags=flags)
        tr.run(stream)
        torch.cuda.synchronize()
        ms = _time_frames(tr, max(1, args.steps if name != "brute" else 2), stream)
        st = tr.stats()
        total = int(np.asarray(st["tests"]).sum()) + int(sum(st["final_tests"]))
        rows[name] = {"ms_per_frame": round(ms, 3), "total_tests": total, "mesh_tests": int(sum(st["mesh_tests"])),
                      "tests_per_ray": round(total / max(1, sum(st["rays"])), 2),
                      "mrays_per_s": round(sum(st["rays"]) / (ms * 1e-3) / 1e6, 3),
                      "by_level": {f"L{k}": int(np.asarray(st["tests"])[:, k].sum()) for k in range(w.levels, 0, -1)},
                      "final_tests": int(sum(st["final_tests"])), "cluster_tests": int(sum(st["cluster_tests"]))}
    bt = rows["brute"]["total_tests"]
    for r in rows.values():
        r["relative_pct"] = round(100.0 * r["total_tests"] / bt, 4)
    rows["crsh_reduction_vs_rah_pct"] = round(100.0 * (1 - rows["crsh"]["total_tests"] / rows["rah"]["total_tests"]), 2)
    for k in ("crsh_zorder", "crsh_objtree", "crsh_zorder_objtree"):
        rows[f"{k}_reduction_vs_rah_pct"] = round(100.0 * (1 - rows[k]["total_tests"] / rows["rah"]["total_tests"]), 2)
    print(json.dumps({"mode": "table4", "workload": w.name, "rays": int(sum(tr.stats()["rays"])), "M": tr.M,
                      "engines": rows}), flush=True)


def run_sweep(args):
    """cfg5 (BASELINE configs[4]): hierarchy depth Lv 2..6 x bundle size B0 in
    {4, 8, 16, 32, 64} at 1024x1024, ~250k triangles in 30 meshes."""
    import torch

    from paper_2312_06538_b200.api import tracer_for
    from workloads import make_workload
    stream = torch.cuda.current_stream()
    base = make_workload(5)
    for lv in (2, 3, 4, 5, 6):
        for b0 in (4, 8, 16, 32, 64):
            base.levels, base.leaf_size, base.branching = lv, b0, 8
            tr = tracer_for(base, flags=7 if args.zorder else 3)
            tr.run(stream)
            torch.cuda.synchronize()
            ms = _time_frames(tr, max(1, args.steps), stream)
            st = tr.stats()
            total = int(np.asarray(st["tests"]).sum()) + int(sum(st["final_tests"]))
            print(json.dumps({"mode": "sweep", "levels": lv, "leaf_size": b0, "branching": 8,
                              "hash": "zorder" if args.zorder else "R6", "ms_per_frame": round(ms, 3),
                              "mrays_per_s": round(sum(st["rays"]) / (ms * 1e-3) / 1e6, 3),
                              "tests_per_ray": round(total / max(1, sum(st["rays"])), 2),
                              "by_level": {f"L{k}": int(np.asarray(st["tests"])[:, k].sum()) for k in range(lv, 0, -1)},
                              "final_tests": int(sum(st["final_tests"])), "cluster_tests": int(sum(st["cluster_tests"]))}), flush=True)
            del tr


def run_whitted(args):
    """Multi-bounce Whitted loop (crsh_render_whitted) on
    the chosen config: rays of all bounces per second, with the oracle's loop
    timed beside it on a band of rows (not the contract line)."""
    import torch

    import oracle
    from paper_2312_06538_b200.api import tracer_for
    from workloads import make_workload
    w = make_workload(args.config)
    flags = 7 if args.zorder else 3
    tr = tracer_for(w, flags=flags)
    stream = torch.cuda.current_stream()
    for _ in range(max(3, args.warmup)):
        img, st = tr.render(w.tri_mat, args.whitted)
    torch.cuda.synchronize()
    ms = []
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    for _ in range(max(1, args.steps)):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        img, st = tr.render(w.tri_mat, args.whitted)
        b.record(stream)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    rays = int(sum(st["rays"]))
    t = float(np.median(ms))
    line = {"mode": "whitted", "metric": "secondary Mrays/s, all bounces of the Whitted loop", "unit": "Mrays/s",
            "value": round(rays / (t * 1e-3) / 1e6, 3), "ms_per_frame": round(t, 3), "depth": args.whitted,
            "hash": "zorder" if args.zorder else "R6", "workload": w.name, "vertices": st["vertices"],
            "rays": st["rays"], "tests": [int(x) for x in st["tests"]], "final_tests": [int(x) for x in st["final_tests"]],
            "image_mean": float(img[:w.P].mean())}
    if not args.no_cpu_baseline:
        import dataclasses
        rows = max(1, w.height // 32)
        r0 = (w.height - rows) // 2
        P = w.width
        band = dataclasses.replace(w, height=rows,
                                   pos=np.ascontiguousarray(w.pos.reshape(3, w.height, P)[:, r0:r0 + rows].reshape(3, -1)),
                                   nrm=np.ascontiguousarray(w.nrm.reshape(3, w.height, P)[:, r0:r0 + rows].reshape(3, -1)),
                                   mat=np.ascontiguousarray(w.mat.reshape(w.height, P)[r0:r0 + rows].reshape(-1)))
        t0 = time.perf_counter()
        ref = oracle.whitted(band, args.whitted, flags=flags)
        dt = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": round(sum(ref["rays"]) / dt / 1e6, 5), "unit": "Mrays/s",
                                "cores": oracle.default_threads(), "kind": "oracle",
                                "sample": f"{rows} of {w.height} image rows (centre band), {sum(ref['rays'])} rays, {dt:.1f} s"}
    print(json.dumps(line), flush=True)


def run_animate(args):
    """Animated scene (the paper's multi-frame averages,
    P:307): every frame moves the object meshes (crsh_scene_transform: a
    rotation about each object's vertical axis plus a bob), renders the
    G-buffer with the GPU primary pass (crsh_primary_gbuffer) and traces the
    secondary rays; the frame time is averaged over the animation (not the
    contract line)."""
    import torch

    import paper_2312_06538_b200 as crsh
    from workloads import make_camera, make_workload
    w = make_workload(args.config)
    flags = 7 if args.zorder else 3
    scene = crsh.Scene(torch.as_tensor(w.tris).cuda(), torch.as_tensor(w.mesh_ids).cuda())
    tm = torch.as_tensor(w.tri_mat).cuda()
    mats = torch.as_tensor(w.materials).cuda()
    cam = make_camera()
    W, H, P = w.width, w.height, w.width * w.height
    opts = crsh.make_opts(w.levels, w.leaf_size, w.branching, flags)
    pos = torch.empty(3 * P, dtype=torch.float32, device="cuda")
    nrm = torch.empty(3 * P, dtype=torch.float32, device="cuda")
    mat = torch.empty(P, dtype=torch.int32, device="cuda")
    ph = torch.empty(P, dtype=torch.int32, device="cuda")
    pt = torch.empty(P, dtype=torch.float32, device="cuda")
    slots = crsh.num_slots(P, w.lights.shape[0], w.ray_types)
    hit = torch.empty(slots, dtype=torch.int32, device="cuda")
    t = torch.empty(slots, dtype=torch.float32, device="cuda")
    hits = crsh.make_hits(W, H, pos, nrm, mat, mats, w.materials.shape[0], w.eye)
    n_m = int(w.mesh_ids.max()) + 1
    tris = w.tris.reshape(-1, 3, 3).astype(np.float64)
    centres = np.stack([tris[w.mesh_ids == m].reshape(-1, 3).mean(0) for m in range(n_m)])
    n_walls = 6

    def xforms(f):
        X = np.zeros((n_m, 12), np.float32)
        for m in range(n_m):
            a = 0.0 if m < n_walls else 2 * np.pi * f / max(1, args.animate) * (1 + m % 3)
            c, s_ = np.cos(a), np.sin(a)
            R = np.array([[c, 0, s_], [0, 1, 0], [-s_, 0, c]])
            b = centres[m] - R @ centres[m] + (0 if m < n_walls else np.array([0, 0.2 * np.sin(a), 0]))
            X[m] = np.concatenate([R, b[:, None]], axis=1).reshape(12)
        return X

    stream = torch.cuda.current_stream()
    ms, rays, tms = [], 0, []
    for f in range(args.animate + 3):
        X = xforms(f)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        crsh.scene_transform(scene, X)
        t1 = time.perf_counter()
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record(stream)
        crsh.primary_gbuffer(scene, cam, W, H, tm, opts, pos, nrm, mat, ph, pt, stream.cuda_stream)
        crsh.trace_secondary(scene, hits, w.lights, w.ray_types, opts, hit, t, stream.cuda_stream)
        b_.record(stream)
        torch.cuda.synchronize()
        if f >= 3:
            ms.append(a_.elapsed_time(b_))
            tms.append((t1 - t0) * 1e3)
            rays += int(sum(crsh.stats(scene)["rays"]))
    line = {"mode": "animate", "metric": "secondary Mrays/s averaged over an animation (moving meshes, GPU primary pass)",
            "unit": "Mrays/s", "value": round(rays / (sum(ms) * 1e-3) / 1e6, 3), "frames": args.animate,
            "ms_per_frame_primary_plus_secondary": round(float(np.mean(ms)), 3),
            "ms_per_frame_transform_host_wall": round(float(np.mean(tms)), 3), "primary_rays_per_frame": P,
            "secondary_rays_per_frame": rays // max(1, len(ms)), "hash": "zorder" if args.zorder else "R6",
            "workload": w.name}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4, help="BASELINE.json configs[N-1]; 4 = the metric's 1920x1080 "
                                                                 "headline workload")
    ap.add_argument("--impl", default="crsh", choices=["crsh", "reference"])
    ap.add_argument("--zorder", action="store_true", help="Z-order hash layout (SURVEY §8(f) NEXT-4)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--nccl-merge", action="store_true", help="N > 1: NCCL MIN all-reduce merge instead of the fused peer stores")
    ap.add_argument("--single-hash", action="store_true", help="skip the second hash layout's extra keys")
    ap.add_argument("--objtree", action="store_true", help="object sphere-tree below the mesh spheres (NEXT-4)")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the N > 1 path (crsh_dist_init, in-library merge) even at N = 1 (tests)")
    ap.add_argument("--table4", action="store_true", help="CRSH vs RAH vs N x M report (not the contract line)")
    ap.add_argument("--sweep", action="store_true", help="cfg5 depth/bundle sweep (not the contract line)")
    ap.add_argument("--whitted", type=int, default=None, metavar="D",
                    help="multi-bounce Whitted loop of depth D (NEXT-2; not the contract line)")
    ap.add_argument("--animate", type=int, default=None, metavar="F",
                    help="F animated frames: moving meshes + GPU primary pass + secondary trace (NEXT-3)")
    args = ap.parse_args()
    if args.animate is not None:
        return run_animate(args)
    if args.whitted is not None:
        return run_whitted(args)
    if args.table4:
        return run_table4(args)
    if args.sweep:
        return run_sweep(args)
    if args.warmup < 3:
        args.warmup = 3
    if args.nccl_merge:
        os.environ["CRSH_DIST_MERGE"] = "nccl"
    if args.impl == "reference":
        run_reference(args)
    else:
        run_crsh(args)


if __name__ == "__main__":
    main()
