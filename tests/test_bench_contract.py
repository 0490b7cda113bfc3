"""The bench.py JSON line contract (task spec): one line with metric / value /
unit / n_gpus / steps / warmup / ms_per_step / higher_is_better / scaling /
vs_baseline / dtype / data / config.workload, plus roofline, cpu_baseline,
e2e, gpu_launches and clocks; the reference arm's line; the CLI's warm-up
floor. GPU for the product arm; the reference arm runs the oracle on the host."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def _common(d):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"):
        assert k in d, k
    assert d["warmup"] >= 3 and d["higher_is_better"] is True and d["scaling"] in ("weak", "strong")
    assert "workload" in d["config"]
    assert d["value"] > 0 and d["ms_per_step"] > 0


@pytest.mark.gpu
def test_product_line():
    d = _run("--steps", "3", "--warmup", "1")   # warm-up floor: raised to 3
    _common(d)
    assert d["warmup"] == 3 and d["n_gpus"] == 1 and d["steps"] == 3
    r = d["roofline"]
    assert r["bound"] in ("alu", "hbm", "tensor") and 0 < r["frac"] <= 1 and r["achieved"] > 0 and r["peak"] > 0
    assert d["gpu_launches"] > 0
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(d["e2e"])
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


def test_reference_line_on_host():
    """--impl reference times the oracle as it stands on the host cores (no GPU needed)."""
    d = _run("--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "3")
    _common(d)
    assert d["impl"] == "reference"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
@pytest.mark.parametrize("mode,name", [("peer", "fused-peer-stores"), ("nccl", "nccl-allreduce-min")])
def test_product_line_dist_path(mode, name, monkeypatch):
    """The N > 1 code path of bench.py (gloo host group, crsh_dist_init, the
    library's merge inside every timed frame) with a world-1 NCCL communicator:
    the line reports the merge that ran, and the merged frame equals the
    rank's own world-1 frame bit for bit."""
    monkeypatch.setenv("CRSH_DIST_MERGE", mode)
    d = _run("--force-dist", "--config", "2", "--single-hash", "--no-cpu-baseline", "--steps", "3")
    assert d["config"]["merge"] == name
    assert d["merge_check"] == "merged frame == world-1 frame on every rank"
    assert d["value"] > 0 and d["e2e"]["value"] > 0
