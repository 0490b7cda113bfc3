#!/usr/bin/env python
"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck), one
tool per gpurun call (B200_PROFILING.md): the smoke() frame (64x64, SH+RE+RR,
2 lights, cfg1 scene, checked against the oracle) and one 128x128 cfg2 frame
per flag set (R6, Z-order, Z-order + object tree) with CRSH_NO_GRAPH=1 so
every kernel is an ordinary launch, also checked against the oracle."""
import os
import sys

os.environ.setdefault("CRSH_NO_GRAPH", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import __graft_entry__  # noqa: E402
import oracle  # noqa: E402
from paper_2312_06538_b200.api import tracer_for  # noqa: E402
from workloads import make_workload  # noqa: E402

__graft_entry__.smoke()
w = make_workload(2, width=128, height=128)
for flags in (3, 7, 71):
    tr = tracer_for(w, flags=flags)
    tr.run()
    hit, t = tr.results()
    ref = oracle.trace(w, flags=flags)
    assert np.array_equal(hit, ref["hit_tri"]) and np.array_equal(t, ref["t"]), flags
    print(f"cfg2 128x128 flags {flags}: ok, {tr.launches()} launches", flush=True)
print("sanitize case done")
