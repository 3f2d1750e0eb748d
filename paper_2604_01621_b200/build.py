"""In-tree build of libdwdp.so (sm_100a CUDA kernels + C++ host runtime + C-ABI).

    python -m paper_2604_01621_b200.build      # incremental

nvcc cross-compiles for sm_100a without a GPU; the .so lands next to this file
so it travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libdwdp.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")

CU = ["kernels.cu", "gemm_sm100.cu", "attn_sm100.cu"]
CPP = ["plan.cpp", "report.cpp", "runtime.cpp", "dep.cpp", "capi.cpp", "mla.cpp"]
HEADERS = ["kernels.hpp", "gemm_sm100.hpp", "plan.hpp", "runtime.hpp", "report.hpp", "attn_sm100.hpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _newer(src: list[str], dst: str) -> bool:
    if not os.path.exists(dst):
        return True
    t = os.path.getmtime(dst)
    return any(os.path.getmtime(s) > t for s in src)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {os.path.basename(cmd[-1])}")


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    deps = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "dwdp.h")]
    objs = []
    for f in CU:
        src, obj = os.path.join(CSRC, f), os.path.join(OBJ, f + ".o")
        objs.append(obj)
        if _newer([src, *deps], obj):
            _run([NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
                  "-Xptxas", "-v" if verbose else "-O3", "-c", src, "-o", obj])
    for f in CPP:
        src, obj = os.path.join(CSRC, f), os.path.join(OBJ, f + ".o")
        objs.append(obj)
        if _newer([src, *deps], obj):
            _run(["g++", "-O2", "-std=c++17", "-fPIC", "-Wall", "-Wextra", "-ffp-contract=off",
                  f"-I{CUDA}/include", "-c", src, "-o", obj])
    if _newer(objs, LIB):
        _run(["g++", "-shared", "-o", LIB, *objs, f"-L{CUDA}/lib64", "-lcudart_static", "-lrt",
              "-lpthread", "-ldl", "-Wl,--exclude-libs,ALL"])
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
