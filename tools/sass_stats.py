#!/usr/bin/env python
"""Per-kernel SASS statistics of a built library: instructions, local-memory
spills (LDL/STL), calls. Usage: python tools/sass_stats.py lib.so [regex]"""
import re
import subprocess
import sys

lib = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
for f in re.split(r"\n\s*Function : ", sass)[1:]:
    name = f.split("\n", 1)[0].strip()
    if pat and not pat.search(name):
        continue
    ins = re.findall(r"/\*[0-9a-f]{4,}\*/\s+([^;]+);", f)
    ops = [i.split()[0] if not i.startswith("@") else i.split()[1] for i in ins]
    cnt = lambda p: sum(1 for o in ops if o.startswith(p))  # noqa: E731
    print(f"{name[:70]:70s} inst {len(ops):6d} LDL {cnt('LDL'):4d} STL {cnt('STL'):4d} CALL {cnt('CALL'):3d}")
