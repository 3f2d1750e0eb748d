"""The drop-in boundary on the GPU from C++ alone: tests/cpp/dwdp_gpu_probe.cpp
(reference-named adapter include/dwdp.hpp + C-ABI, CUDA driver API for the
buffers, no Python/torch on its path) runs two DWDP ranks against the
all-local model; outputs must be bitwise equal."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cpp_host_dwdp_layers_match_all_local(tmp_path):
    from paper_2604_01621_b200._lib import LIB_PATH, lib
    lib()
    exe = str(tmp_path / "dwdp_gpu_probe")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                        f"-I{cuda}/include", os.path.join(ROOT, "tests", "cpp", "dwdp_gpu_probe.cpp"),
                        LIB_PATH, f"-L{cuda}/lib64/stubs", "-lcuda",
                        f"-Wl,-rpath,{os.path.dirname(LIB_PATH)}", "-o", exe],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    lines = out.stdout.splitlines()
    assert sum(1 for ln in lines if ln.startswith("L ") and ln.endswith("bitwise-equal")) == 8
    recs = [ln for ln in lines if ln.startswith("R ")]
    assert len(recs) == 2 and all("prefetch_bytes=" in ln and not ln.endswith("=-1") for ln in recs)
