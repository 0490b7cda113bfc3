"""Debug: per-level tests/hits of the GPU build vs the oracle for one config."""
import sys
import numpy as np
sys.path.insert(0, '.')
import oracle
import paper_2312_06538_b200 as crsh
from paper_2312_06538_b200.api import tracer_for
from workloads import make_workload
w = make_workload(2, width=96, height=96, levels=3, leaf_size=4, branching=4)
tr = tracer_for(w)
tr.run()
hit, t = tr.results()
st = crsh.stats(tr.scene)
ref = oracle.trace(w)
print('hits equal', np.array_equal(hit, ref['hit_tri']))
for seg in range(3):
    print(seg, 'gpu tests', st['tests'][seg][:4], 'hits', st['hits'][seg][:4])
    print(seg, 'ora tests', ref['stats']['tests'][seg][:4], 'hits', ref['stats']['hits'][seg][:4])
