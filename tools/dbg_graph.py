import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2312_06538_b200 as crsh
from paper_2312_06538_b200.api import tracer_for
from workloads import make_workload
w = make_workload(2)
tr = tracer_for(w, flags=3 | crsh.F_STAGE_TIMING)
for i in range(3):
    tr.run(); st = tr.stats(); print('stage', st['stage_ms'])
import ctypes
L = crsh.load()
hh = np.empty(tr.slots, np.int32); ht = np.empty(tr.slots, np.float32)
tr.run_host(np.ascontiguousarray(w.pos), np.ascontiguousarray(w.nrm), np.ascontiguousarray(w.mat), np.ascontiguousarray(w.materials), hh, ht)
h, t = tr.results()
print('host==dev', np.array_equal(hh, h))
