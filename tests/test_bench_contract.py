"""bench.py's JSON-line contract (the driver parses it): a short N=1 run of
the real bench and of the reference arm, checked key by key."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

BASE = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config"]


def _run(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                       text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_has_every_contract_key():
    d = _run("--steps", "2", "--warmup", "3", "--layers", "2", "--tokens", "8192",
             "--cpu-tokens", "4")
    for k in BASE + ["roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"]:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["value"] > 0
    assert d["config"]["workload"]
    rf = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in rf, k
    assert 0 < rf["frac"] < 1.5
    cb = d["cpu_baseline"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in cb, k
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert d["step_roofline"]["frac"] > 0
    assert d["report"]["dwdp"]["iteration_latency_us"] > 0


def test_reference_arm_line():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "1", "--ref-tokens", "2",
             "--layers", "2")
    assert d["impl"] == "reference"
    for k in BASE + ["cpu_baseline", "e2e"]:
        assert k in d, k
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["cores"] >= 1


def test_bench_line_nvfp4_and_attention():
    """The NVFP4 arm (measured-ratio peak, nvfp4 dtype label) and the attention
    window keep the same contract."""
    d = _run("--steps", "2", "--warmup", "3", "--layers", "2", "--tokens", "8192", "--dtype", "nvfp4",
             "--attention", "--no-cpu-baseline")
    assert d["dtype"].startswith("nvfp4") and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["unit"] == "TFLOP/s" and 0 < d["roofline"]["frac"] < 1.5
    assert d["attention"]["ms_per_layer"] > 0 and d["config"]["attention_block"] is True
