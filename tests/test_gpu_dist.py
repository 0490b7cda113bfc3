"""The library's NCCL data plane (crsh_dist_init, csrc/dist.cuh; SURVEY §8(a)
a14, §8(b), §8(e)) on one GPU: a world-1 NCCL communicator, so every step of
the merge runs -- the symmetric window (ncclMemAlloc + ncclCommWindowRegister),
the LSA pointers resolved on the device, the fused peer stores of the
epilogue, both LSA barriers, the unpack from the window, the ncclAllReduce of
the counters -- or, with CRSH_DIST_MERGE=nccl, the ncclAllReduce(MIN) merge of
the packed frame.  The merged frame and the summed counters must equal the
oracle's.  (NCCL refuses two ranks on one GPU, so a world-2 exchange cannot
run here; tests/test_gpu_two_process.py merges two real ranks over gloo.)
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, json
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2312_06538_b200 as crsh
from paper_2312_06538_b200 import dist
from paper_2312_06538_b200.api import tracer_for
from workloads import make_workload
import oracle
w = make_workload(2, width=256, height=256)
out = {}
for flags in (3, 7):
    tr = tracer_for(w, flags=flags)
    dist.init(tr.scene, dist.unique_id(), 0, 1)
    try:
        dist.init(tr.scene, dist.unique_id(), 0, 1)
        second = "accepted"
    except crsh.CrshError as e:
        second = e.status
    for rep in range(3):      # capture, then graph replays
        tr.run()
        hit, t = tr.results()
        st = crsh.stats(tr.scene)
    ref = oracle.trace(w, flags=flags)
    rs = ref["stats"]
    ok = bool(np.array_equal(hit, ref["hit_tri"]) and np.array_equal(t.view(np.uint32), ref["t"].view(np.uint32)))
    cnt = all(np.array_equal(st[k], rs[k]) for k in ("tests", "hits")) and all(
        list(st[k]) == list(rs[k]) for k in ("mesh_tests", "mesh_hits", "final_tests", "final_hits", "rays_hit", "rays"))
    # the explicit sharded API is unaffected by dist (no merge)
    import torch
    packed = torch.empty(tr.slots, dtype=torch.int64, device="cuda")
    tr.run_packed(packed)
    torch.cuda.synchronize()
    bad = crsh.make_opts(2, 8, 8, flags, 0, 2)
    try:
        crsh.trace_secondary(tr.scene, tr.hits, w.lights, w.ray_types, bad, tr.hit_tri, tr.t)
        mismatch = "accepted"
    except crsh.CrshError as e:
        mismatch = e.status
    out[flags] = dict(hits_equal=ok, counts_equal=bool(cnt), merge=st["merge"], second=second, mismatch=mismatch,
                      launches=tr.launches())
# window growth (a collective re-registration) and the host-buffer call on a dist scene
tr = tracer_for(make_workload(2, width=64, height=64), flags=3)
dist.init(tr.scene, dist.unique_id(), 0, 1)
tr.run()
small_ok = bool(np.array_equal(tr.results()[0], oracle.trace(make_workload(2, width=64, height=64))["hit_tri"]))
w2 = make_workload(2, width=160, height=120)
tr.set_gbuffer(w2.width, w2.height, w2.pos, w2.nrm, w2.mat, w2.materials, w2.eye)
tr.configure(w2.lights, w2.ray_types, w2.levels, w2.leaf_size, w2.branching, 3)
tr.run()
ref2 = oracle.trace(w2)
grow_ok = bool(np.array_equal(tr.results()[0], ref2["hit_tri"]))
hh = np.empty(tr.slots, np.int32); th = np.empty(tr.slots, np.float32)
tr.run_host(np.ascontiguousarray(w2.pos), np.ascontiguousarray(w2.nrm), np.ascontiguousarray(w2.mat),
            np.ascontiguousarray(w2.materials), hh, th)
host_ok = bool(np.array_equal(hh, ref2["hit_tri"]) and np.array_equal(th.view(np.uint32), ref2["t"].view(np.uint32)))
errs = []
for args in ((0, 0), (1, 1), (-1, 1)):
    t3 = tracer_for(make_workload(1, width=8, height=8))
    try:
        dist.init(t3.scene, dist.unique_id(), *args)
        errs.append("accepted")
    except crsh.CrshError as e:
        errs.append(e.status)
out["extra"] = dict(small=small_ok, grow=grow_ok, host=host_ok, bad_rank_world=errs)
print("RESULT " + json.dumps(out))
'''


@pytest.mark.parametrize("mode,code", [("peer", 2), ("nccl", 1)])
def test_dist_world1_merge_equals_oracle(mode, code):
    env = dict(os.environ, CRSH_DIST_MERGE=mode, NCCL_DEBUG="WARN")
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT], capture_output=True, text=True, env=env, timeout=900)
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT ")]
    assert r.returncode == 0 and line, r.stdout[-3000:] + r.stderr[-3000:]
    import json
    res = json.loads(line[0][7:])
    extra = res.pop("extra")
    assert extra["small"] and extra["grow"] and extra["host"], extra
    assert extra["bad_rank_world"] == [2, 2, 2], extra   # EINVAL before any NCCL call
    for flags, v in res.items():
        assert v["hits_equal"], (mode, flags)
        assert v["counts_equal"], (mode, flags)
        assert v["merge"] == code, (mode, flags, v["merge"])
        assert v["second"] == 2 and v["mismatch"] == 2, v   # EINVAL
        assert v["launches"] > 0
