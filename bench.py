#!/usr/bin/env python
"""bench.py -- secondary Mrays/s of the CRSH path (BASELINE.json metric).

One step = one frame of the whole hot path through the C
ABI call crsh_trace_secondary: generate + hash + trim, compress, radix sort,
decompress, build, mesh cull, traversal, final tests, per-slot output (plus,
at N > 1, the NCCL min-merge of the per-rank packed results).

Default workload: BASELINE.json configs[1] ("512x512 shadow+reflection rays,
~70k-triangle multi-mesh procedural scene, 1 B200"), seeded synthetic scene +
rasterised G-buffer (workloads/).  Timing: W untimed warm-up frames, then K
frames, each bracketed by CUDA events on the launching stream after an L2
flush (a 512 MiB write outside the bracket); barrier + synchronize on both
sides; max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl crsh|reference]
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


def trav_flops(st):
    return int(np.asarray(st["tests"]).sum()) * EQ9_FLOPS + int(sum(st["final_tests"])) * MT_FLOPS


def load_traffic(config, zorder, kernel="k_traverse"):
    """DRAM bytes per launch of `kernel` from the committed ncu launch list of
    the same workload (profiles/ncu_summary*.json: cfg2, R6 or Z-order);
    null for workloads without a committed capture."""
    if config != 2:
        return None
    p = os.path.join(ROOT, "profiles", "ncu_summary_zorder.json" if zorder else "ncu_summary.json")
    try:
        d = json.load(open(p))
        return d.get("kernels", {}).get(kernel, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


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


def oracle_sample(w, flags, target_s=12.0):
    """Grow a centre band of image rows until one oracle run takes about
    target_s seconds of host CPU work (or the whole image); returns (rays,
    seconds, rows, cores)."""
    import oracle
    prep = oracle.ScenePrep(w.tris, w.mesh_ids)
    rows = max(1, w.height // 64)
    while True:
        rays, dt = oracle_band(w, flags, rows, prep)
        if dt >= target_s / 4 or rows >= w.height:
            return rays, dt, rows, oracle.default_threads()
        rows = min(w.height, max(rows + 1, int(rows * min(8.0, target_s / max(dt, 1e-3)))))


# ----------------------------------------------------------------------------- GPU arm
def run_crsh(args):
    import torch
    import torch.distributed as dist

    import paper_2312_06538_b200 as crsh
    from paper_2312_06538_b200.api import tracer_for
    from workloads import make_workload

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    flags = crsh.F_SORT | crsh.F_MESH_CULL | (crsh.F_ZORDER if args.zorder else 0)
    w = make_workload(args.config)
    tr = tracer_for(w, device=local, flags=flags | crsh.F_KERNEL_TIMING, shard_rank=rank, shard_world=world)
    stream = torch.cuda.current_stream()
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    packed = torch.empty(max(tr.slots, 1), dtype=torch.int64, device="cuda") if world > 1 else None
    # N > 1 merge: the fused epilogue stores each rank's owned
    # results straight into every rank's symmetric window over NVLink
    # (crsh_trace_secondary_peer), bracketed by device-side barriers; checked
    # once against the NCCL MIN all-reduce merge, which it replaces (and which
    # stays the path if the symmetric window is unavailable or disagrees).
    merge, hdl, ptrs, sbuf = ("none" if world == 1 else "nccl"), None, None, None
    if world > 1 and not args.nccl_merge:
        # every rank allocates first and the ranks agree before the collective
        # rendezvous, so one rank's failure cannot leave the others waiting in it
        try:
            import torch.distributed._symmetric_memory as symm_mem
            sbuf = symm_mem.empty(max(tr.slots, 1), dtype=torch.int64, device=torch.device("cuda", local))
            ok_alloc = 1
        except Exception as e:
            print(f"[bench] symmetric allocation failed ({type(e).__name__}: {e})", file=sys.stderr)
            ok_alloc = 0
        flag = torch.tensor([ok_alloc], dtype=torch.int32, device="cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if world > 1 and not args.nccl_merge and int(flag) == 1:
        try:
            hdl = symm_mem.rendezvous(sbuf, dist.group.WORLD)
            ptrs = [int(hdl.buffer_ptrs[r]) for r in range(world)]
            hdl.barrier()
            tr.run_peer(ptrs, stream)
            hdl.barrier()
            tr.run_packed(packed, stream)
            dist.all_reduce(packed, op=dist.ReduceOp.MIN)
            ok = torch.tensor([1 if torch.equal(sbuf, packed) else 0], dtype=torch.int32, device="cuda")
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            merge = "peer" if int(ok) == 1 else "nccl"
        except Exception as e:   # no P2P / symmetric memory on this box: keep the NCCL merge
            print(f"[bench] fused peer merge unavailable ({type(e).__name__}: {e}); NCCL all-reduce merge", file=sys.stderr)
            merge = "nccl"

    def step():
        if world == 1:
            tr.run(stream)
        elif merge == "peer":
            hdl.barrier()                      # every rank done reading the previous frame
            tr.run_peer(ptrs, stream)          # owned results -> every rank's window
            hdl.barrier()                      # all stores landed
            tr.unpack(sbuf, stream)
        else:
            tr.run_packed(packed, stream)
            dist.all_reduce(packed, op=dist.ReduceOp.MIN)   # per-slot min-merge over NVLink
            tr.unpack(packed, stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    st0 = tr.stats()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    stage = np.zeros(8)
    launches = 0
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
            st = tr.stats()          # synchronises; outside the event bracket
            stage += np.asarray(st["stage_ms"])
            launches += tr.launches() + (1 if world > 1 else 0)   # + the unpack kernel
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms = np.array([a.elapsed_time(b) for a, b in ev])
    total_ms = float(ms.sum())
    trav_ms = stage[6] / args.steps
    # per-stage breakdown (diagnostic, outside the timed region): same frames with all stage events
    trs = tracer_for(w, device=local, flags=flags | crsh.F_STAGE_TIMING, shard_rank=rank, shard_world=world)
    stage = np.zeros(8)
    n_diag = 3
    for _ in range(n_diag + 1):
        if world == 1:
            trs.run(stream)
        else:
            trs.run_packed(packed, stream)
            dist.all_reduce(packed, op=dist.ReduceOp.MIN)
            trs.unpack(packed, stream)
        s_ = trs.stats()
        if _ > 0:
            stage += np.asarray(s_["stage_ms"])
    stage *= args.steps / n_diag
    del trs
    st = tr.stats()
    # counters: traversal counters are per rank (sum); ray counts are global
    vec = torch.tensor([total_ms, trav_ms], dtype=torch.float64, device="cuda")
    cnt = torch.tensor([int(np.asarray(st["tests"]).sum()), int(sum(st["final_tests"])), int(sum(st["mesh_tests"]))],
                       dtype=torch.int64, device="cuda")
    if world > 1:
        dist.all_reduce(vec, op=dist.ReduceOp.MAX)
        dist.all_reduce(cnt, op=dist.ReduceOp.SUM)
    total_ms, trav_ms_max = float(vec[0]), float(vec[1])
    tests_all, final_all, mesh_all = (int(x) for x in cnt.tolist())
    rays = int(sum(st["rays"]))
    mrays = rays * args.steps / (total_ms * 1e-3) / 1e6
    # end to end through the public API with HOST buffers (crsh_trace_secondary_host), N = 1 path
    e2e = None
    if world == 1:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
        hpos, hnrm, hmat, hmats = pin(w.pos), pin(w.nrm), pin(w.mat), pin(w.materials)
        hh = torch.empty(tr.slots, dtype=torch.int32).pin_memory()
        ht = torch.empty(tr.slots, dtype=torch.float32).pin_memory()
        for _ in range(2):
            tr.run_host(hpos.numpy(), hnrm.numpy(), hmat.numpy(), hmats.numpy(), hh.numpy(), ht.numpy(), stream)
        e_ms = []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            tr.run_host(hpos.numpy(), hnrm.numpy(), hmat.numpy(), hmats.numpy(), hh.numpy(), ht.numpy(), stream)
            b.record(stream)
            torch.cuda.synchronize()
            e_ms.append(a.elapsed_time(b))
        P = w.width * w.height
        e2e = {"value": round(rays * len(e_ms) / (sum(e_ms) * 1e-3) / 1e6, 3), "unit": "Mrays/s",
               "h2d_bytes_per_step": 28 * P + 12 * int(w.materials.shape[0]), "d2h_bytes_per_step": 8 * tr.slots,
               "api": "crsh_trace_secondary_host"}
    if rank != 0:
        if world > 1:
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
    tflops = trav_flops(st) / (trav_ms * 1e-3) / 1e12 if trav_ms > 0 else 0.0
    traffic = load_traffic(args.config, args.zorder)
    brute = rays * tr.M
    stage_names = ["generate+trim", "compress", "sort", "decompress", "build", "mesh-cull+plan", "traverse+final",
                   "output"]
    out = {
        "metric": METRIC, "value": round(mrays, 3), "unit": "Mrays/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded procedural scene + rasterised G-buffer, workloads/)",
        "config": {"workload": w.name, "pixels": w.width * w.height, "triangles": tr.M, "meshes": int(w.n_meshes),
                   "ray_types": w.ray_types, "lights": int(w.lights.shape[0]), "levels": w.levels,
                   "leaf_size": w.leaf_size, "branching": w.branching, "hash": "zorder" if args.zorder else "R6 (SPEC layout)",
                   "parallelism": f"hash-range shard x{world}" if world > 1 else "single GPU",
                   "merge": {"none": "none (1 GPU)", "peer": "fused peer stores into symmetric windows (NVLink)",
                             "nccl": "NCCL MIN all-reduce"}[merge],
                   "l2": "flushed before every timed step (512 MiB write outside the event bracket)"},
        "rays_per_step": rays,
        "tests_per_ray": round((tests_all + final_all) / max(rays, 1), 2),
        "tests_by_level": {f"L{k}": int(np.asarray(st["tests"])[:, k].sum()) for k in range(w.levels, 0, -1)},
        "hits_by_level": {f"L{k}": int(np.asarray(st["hits"])[:, k].sum()) for k in range(w.levels, 0, -1)},
        "final_tests": final_all, "mesh_tests": mesh_all,
        "naive_tests_per_ray": tr.M,
        "relative_pct_of_brute": round(100.0 * (tests_all + final_all) / max(brute, 1), 4),
        "stage_ms": {n: round(v / args.steps, 4) for n, v in zip(stage_names, stage)},
        "roofline": {"bound": "alu", "kernel": "k_traverse", "achieved": round(tflops, 3), "peak": round(peak_tflops, 2),
                     "unit": "TFLOP/s", "frac": round(tflops / peak_tflops, 4), "traffic": traffic,
                     "note": f"FP32: {EQ9_FLOPS} flops per Eq 9 test, {MT_FLOPS} per MT test; peak: {peak_src}; "
                             f"kernel time from CUDA events around k_traverse"},
        "gpu_launches": launches,
        "e2e": e2e,
        "paper_context": paper_context(),
        "clocks": clocks,
    }
    if world == 1 and not args.no_cpu_baseline:
        cr, cs, rows, cores = oracle_sample(w, flags & 7)
        out["cpu_baseline"] = {"value": round(cr / cs / 1e6, 5), "unit": "Mrays/s", "cores": cores, "kind": "oracle",
                               "sample": f"{rows} of {w.height} image rows (centre band), {cr} rays, {cs:.1f} s"}
    print(json.dumps(out), flush=True)
    if world > 1:
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
    flags = 3 | (4 if args.zorder else 0)
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
           "config": {"workload": w.name},
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
    for name, flags in (("brute", crsh.F_BRUTE), ("rah", 0), ("crsh", 3), ("crsh_zorder", 7)):
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
                      "final_tests": int(sum(st["final_tests"]))}
    bt = rows["brute"]["total_tests"]
    for r in rows.values():
        r["relative_pct"] = round(100.0 * r["total_tests"] / bt, 4)
    rows["crsh_reduction_vs_rah_pct"] = round(100.0 * (1 - rows["crsh"]["total_tests"] / rows["rah"]["total_tests"]), 2)
    rows["crsh_zorder_reduction_vs_rah_pct"] = round(
        100.0 * (1 - rows["crsh_zorder"]["total_tests"] / rows["rah"]["total_tests"]), 2)
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
                              "final_tests": int(sum(st["final_tests"]))}), flush=True)
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
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="crsh", choices=["crsh", "reference"])
    ap.add_argument("--zorder", action="store_true", help="Z-order hash layout (SURVEY §8(f) NEXT-4)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--nccl-merge", action="store_true", help="N > 1: NCCL MIN all-reduce merge instead of the fused peer stores")
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
    if args.impl == "reference":
        run_reference(args)
    else:
        run_crsh(args)


if __name__ == "__main__":
    main()
