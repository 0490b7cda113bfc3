#!/usr/bin/env python
"""Library yardsticks for the HBM stages a1-a8 (NOT product code; VERDICT r1
"Next round" 4: ">= 70 % of the HBM roofline, or a measured ceiling
argument"). One cfg4 frame runs through libcrsh with stage timing; its own
intermediate data (the chunk keys the sort sorts, the sorted slot permutation
the leaf build gathers by, the chunk run lengths the decompression expands)
is pulled through the debug taps, and PyTorch's library kernels (CUB radix
sort, index_select gather, repeat_interleave, unique_consecutive, a copy) are
timed on the same data with CUDA events, L2 flushed before each, median of
10. Each line: our stage, the library's closest operation on the same data,
and the streaming copy of the stage's SURVEY-model bytes (its roofline).

Usage: python tools/stage_yardsticks.py [--config 4] [--zorder]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2312_06538_b200 as crsh  # noqa: E402
from paper_2312_06538_b200.api import tracer_for  # noqa: E402
from workloads import make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--zorder", action="store_true")
a = ap.parse_args()

dev = torch.device("cuda:0")
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)


def timed(fn, reps=10):
    out = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return float(np.median(out))


w = make_workload(a.config)
flags = crsh.F_SORT | crsh.F_MESH_CULL | (crsh.F_ZORDER if a.zorder else 0)
tr = tracer_for(w, flags=flags | crsh.F_STAGE_TIMING)
stage = np.zeros(8)
for k in range(4):
    flush.zero_()
    tr.run()
    st = tr.stats()
    if k:
        stage += np.asarray(st["stage_ms"]) / 3
ours = dict(zip(crsh.STAGES, stage.tolist()))
segs = [s for s in range(len(st["rays"])) if st["rays"][s] > 0]
ck = np.concatenate([crsh.debug_tap(tr.scene, crsh.TAP_CHUNK_KEYS, s) for s in segs]).astype(np.int64)
cb = [crsh.debug_tap(tr.scene, crsh.TAP_CHUNK_BASE, s).astype(np.int64) for s in segs]
sl = np.concatenate([crsh.debug_tap(tr.scene, crsh.TAP_SORTED_SLOTS, s) for s in segs]).astype(np.int64)
kseg = [crsh.debug_tap(tr.scene, crsh.TAP_KEYS, s) for s in segs]
keys = np.concatenate(kseg).astype(np.int64)
rays = int(sum(st["rays"]))
slots = int(sl.max()) + 1
n_chunks = int(ck.size)
# chunk run lengths: bases are compacted positions relative to the segment
lens = np.concatenate([np.diff(np.append(b, k.size)) for b, k in zip(cb, kseg)])
del tr

t_ck = torch.from_numpy(ck.astype(np.int32)).to(dev)
t_sl = torch.from_numpy(sl).to(dev)
t_keys = torch.from_numpy(keys.astype(np.int32)).to(dev)
t_rays = torch.randn(slots, 8, device=dev)                 # 32-byte ray records by slot
t_base = torch.arange(n_chunks, dtype=torch.int32, device=dev)
t_len = torch.from_numpy(lens).to(dev)
res = {}
res["sort"] = timed(lambda: torch.sort(t_ck, stable=True))            # CUB onesweep, pairs (key, index)
# the leaf build's gather of 32-B rays: the fastest of three library gathers
t_idx8 = t_sl.view(-1, 1).expand(-1, 8)
gathers = {"index_select": lambda: t_rays.index_select(0, t_sl), "advanced indexing": lambda: t_rays[t_sl],
           "gather": lambda: torch.gather(t_rays, 0, t_idx8)}
g_ms = {k: timed(f) for k, f in gathers.items()}
res["build"] = min(g_ms.values())
res["decompress"] = timed(lambda: torch.repeat_interleave(t_base, t_len))
res["compress"] = timed(lambda: torch.unique_consecutive(t_keys, return_counts=True))


def copy_ms(nbytes):
    src = torch.empty(int(nbytes), dtype=torch.uint8, device=dev)
    dst = torch.empty_like(src)
    return timed(lambda: dst.copy_(src))


P = w.width * w.height
c = n_chunks / max(rays, 1)
model_bytes = 28 * P + (120 + 88 * c + 64 / w.leaf_size) * rays   # SURVEY §8(d), as bench.py
a18 = sum(ours[k] for k in ("generate+trim", "compress", "sort", "decompress", "build"))
out = {"workload": w.name, "hash": "zorder" if a.zorder else "R6", "rays": rays, "slots": slots,
       "chunks": n_chunks, "ours_ms": {k: round(v, 4) for k, v in ours.items()},
       "library_ms": {k: round(v, 4) for k, v in res.items()},
       "library_ops": {"sort": "torch.sort(chunk keys, stable) -> CUB radix sort pairs",
                       "build": "gather of 32-B ray records by the sorted slot permutation (fastest of "
                                + ", ".join(f"{k} {v:.3f} ms" for k, v in g_ms.items()) + ")",
                       "decompress": "repeat_interleave(chunk ids, run lengths)",
                       "compress": "unique_consecutive(keys, return_counts)"},
       "a1_a8_ms": round(a18, 4), "model_bytes": int(model_bytes),
       "copy_of_model_bytes_ms": round(copy_ms(model_bytes / 2) , 4),
       "note": "copy_of_model_bytes_ms: a device copy reading and writing model_bytes/2 each (model_bytes moved)"}
print(json.dumps(out))
