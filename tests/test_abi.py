"""CPU checks of the C ABI boundary: libcrsh.so builds for sm_100a, loads, and
exports every function include/crsh.h declares; the product path has no CPU
fallback (it fails loudly without a GPU); host-side logic (slot counts)."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

import paper_2312_06538_b200 as crsh
from paper_2312_06538_b200 import build as nb


@pytest.fixture(scope="module")
def lib():
    nb.build()
    return crsh.load()


def test_exports_every_header_symbol(lib):
    names = crsh.header_functions()
    assert {"crsh_scene_create", "crsh_trace_secondary", "crsh_stats"} <= set(names)
    for n in names:
        assert hasattr(lib, n), n


def test_sm100a_only_and_no_implicit_fma(lib):
    """The cubin is sm_100a (no PTX for JIT to other archs)."""
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", nb.OUT], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    ptx = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-ptx", nb.OUT], capture_output=True, text=True).stdout
    assert ptx.strip() == ""
    assert "--fmad=false" in nb.FLAGS and "--use_fast_math" not in nb.FLAGS


def test_num_slots(lib):
    """Slot count P * (L*[SH] + [RE] + [RR]) (crsh.h, R5)."""
    assert crsh.num_slots(100, 3, 1) == 300
    assert crsh.num_slots(100, 3, 7) == 500
    assert crsh.num_slots(100, 0, 1) == 0
    assert crsh.num_slots(10, 2, 6) == 20


def test_fails_loudly_without_gpu(lib):
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    tris = np.zeros((1, 9), np.float32)
    ids = np.zeros(1, np.int32)
    with pytest.raises(crsh.CrshError) as e:
        crsh.Scene(tris.ctypes.data, ids.ctypes.data, M=1)
    assert e.value.status == 6   # CRSH_ECUDA: no CUDA device, no CPU fallback


def test_invalid_arguments_are_rejected(lib):
    assert lib.crsh_scene_create(None, None, 1, 0, ctypes.byref(ctypes.c_void_p())) == 2
    assert lib.crsh_scene_create(1, 1, 0, 0, ctypes.byref(ctypes.c_void_p())) == 4


def test_product_never_imports_oracle():
    """The product package shares no code with oracle/ (DESIGN.md §2)."""
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pkg = os.path.join(here, "paper_2312_06538_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(root, f)).read()
                assert "import oracle" not in src and "from oracle" not in src and "oracle.cpp" not in src, f


def test_packed_arithmetic_not_contracted():
    """NUMSPEC fixes every rounding: ptxas must not fuse a packed
    multiply into a following add (it does fuse mul.rn.f32x2 + sub.rn.f32x2
    into FFMA2 when the product has a single use, even under --fmad=false).
    Per kernel, the SASS of the built library must hold every FFMA2 / FMUL2 /
    FADD2 the PTX asks for, with no surplus FFMA2 that is not matched by
    duplicated multiplies and adds (block duplication, not fusion)."""
    import re
    import shutil
    import subprocess
    import tempfile
    from paper_2312_06538_b200 import build as nb
    nvcc, cuobjdump = nb.NVCC, shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not (os.path.exists(nvcc) and os.path.exists(cuobjdump)):
        pytest.skip("CUDA toolchain not available")
    lib = nb.build()
    with tempfile.TemporaryDirectory() as d:
        ptx_path = os.path.join(d, "crsh.ptx")
        flags = [f for f in nb.FLAGS if f not in ("-shared", "-Xcompiler", "-fPIC", "-cudart", "static", "-lineinfo")]
        flags += [f for f in nb.nccl_flags() if f.startswith("-I")]
        subprocess.check_call([nvcc, *flags, "-ptx", "-o", ptx_path, nb.SRC])
        ptx = open(ptx_path).read()
    sass = subprocess.run([cuobjdump, "-sass", lib], capture_output=True, text=True).stdout
    want = {}
    for e in re.split(r"\n\.visible \.entry ", ptx)[1:]:
        name = e.split("(", 1)[0]
        want[name] = (len(re.findall(r"fma\.rn\.f32x2", e)), len(re.findall(r"mul\.rn\.f32x2", e)),
                      len(re.findall(r"(?:add|sub)\.rn\.f32x2", e)))
    checked = 0
    for f in re.split(r"\n\s*Function : ", sass)[1:]:
        name = f.split("\n", 1)[0].strip()
        if name in want and sum(want[name]):
            got = (len(re.findall(r"\bFFMA2 ", f)), len(re.findall(r"\bFMUL2 ", f)), len(re.findall(r"\bFADD2 ", f)))
            # ptxas may duplicate whole blocks (e.g. a peeled iteration of
            # the unrolled Eq 9 pairs), which only adds instructions in the
            # blocks' proportions (cull2: 8 FFMA2 : 4 FMUL2 : 4 FADD2, mt2o:
            # 7 : 7 : 0); a fused mul + add/sub instead REMOVES one FMUL2 and
            # one FADD2 and adds an FFMA2. So: nothing the PTX asks for is
            # missing, and any surplus FFMA2 is matched by at least as many
            # surplus FMUL2 + FADD2 (duplicated code), never by fusion.
            dfma, dmul, dadd = (g - w for g, w in zip(got, want[name]))
            assert dfma >= 0 and dmul >= 0 and dadd >= 0, (name, got, want[name])
            assert dfma <= dmul + dadd, (name, got, want[name])
            checked += 1
    assert checked >= 4   # the k_traverse variants at least
