"""The drop-in boundary: libdwdp.so loads (no GPU needed) and exports every
entry point include/dwdp.h declares; the product path has no CPU fallback."""
import os
import re
import subprocess

import pytest

from conftest import ROOT


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "dwdp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dwdp_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert len(syms) >= 40
    for s in ["dwdp_placement_build", "dwdp_copy_plan_build", "dwdp_prefetch_issue",
              "dwdp_moe_forward", "dwdp_layer_forward", "dwdp_stack_forward"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2604_01621_b200._lib import LIB_PATH, SIGNATURES, lib
    L = lib()
    out = subprocess.run(["nm", "-D", "--defined-only", LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (dwdp_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    for s in declared_symbols():
        getattr(L, s)
        assert s in SIGNATURES, f"python binding lacks {s}"


def test_library_is_sm100a_only():
    from paper_2604_01621_b200._lib import LIB_PATH
    out = subprocess.run(["cuobjdump", "--list-elf", LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
    sass = subprocess.run(["cuobjdump", "-sass", LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass  # tcgen05 + TMA + TMEM


def test_errors_map_to_reference_exceptions():
    import paper_2604_01621_b200 as D
    with pytest.raises(D.ConfigError):
        D.build_copy_plan([D.ShardRef(1, 0, 5, 0)], 0, 0)
    from paper_2604_01621_b200._lib import lib
    assert "sm_100a" in lib().dwdp_version().decode()


def test_context_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2604_01621_b200 as D
    with pytest.raises(D.CudaError):
        D.DwdpContext(D.DwdpConfig.tiny())
