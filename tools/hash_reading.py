#!/usr/bin/env python
"""Tests per ray by segment (SH vs RE vs RR) for the R6 and Z-order hashes and
for RAH, from the oracle (the hash-reading question; VERDICT r1
item 8). Usage: python tools/hash_reading.py CFG [WIDTH HEIGHT]"""
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from workloads import make_workload  # noqa: E402

cfg = int(sys.argv[1])
kw = dict(width=int(sys.argv[2]), height=int(sys.argv[3])) if len(sys.argv) > 3 else {}
w = make_workload(cfg, **kw)
prep = oracle.ScenePrep(w.tris, w.mesh_ids)
out = {"workload": w.name, "pixels": w.P, "triangles": int(prep.M)}
for name, fl in (("rah", 0), ("R6", 3), ("zorder", 7), ("R6_objtree", 67), ("zorder_objtree", 71)):
    st = oracle.trace(w, prep, flags=fl)["stats"]
    row = {}
    for seg, label in ((0, "SH"), (1, "RE"), (2, "RR")):
        n = st["rays"][seg]
        if not n:
            continue
        tot = int(np.asarray(st["tests"][seg]).sum()) + int(st["final_tests"][seg])
        row[label] = {"rays": int(n), "tests_per_ray": round(tot / n, 1)}
    out[name] = row
print(json.dumps(out))
