"""Multi-GPU parity: DWDP (IPC peer pulls) and DEP (NCCL all-to-alls) equal
the all-local model bit for bit, one process per GPU (tests/mp_check.py)."""
import os
import subprocess
import sys

import pytest
import torch

from conftest import ROOT

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


@pytest.mark.parametrize("engine,weight", [(0, 0), (1, 0), (2, 0), (1, 1), (0, 1), (1, 2), (0, 2)])
def test_dwdp_and_dep_match_all_local(engine, weight):
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    n = min(n, 4)
    env = dict(os.environ, DWDP_ENGINE=str(engine), DWDP_WEIGHT=str(weight))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={n}", "--master-addr=127.0.0.1",
                        f"--master-port={29600 + 3 * engine + weight}", os.path.join(ROOT, "tests", "mp_check.py")],
                       env=env, capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "failures=0" in out, out[-4000:]


@pytest.mark.parametrize("engine,weight", [(1, 0), (0, 0), (1, 1), (0, 2)])
def test_dwdp_and_dep_match_all_local_r1_shapes(engine, weight):
    """BASELINE config 3 shapes (R1 layer, 88 MB bf16 experts) over real CUDA
    IPC pulls: DWDP and DEP layers bit-identical to the all-local model."""
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    n = min(n, 4)
    env = dict(os.environ, DWDP_ENGINE=str(engine), DWDP_WEIGHT=str(weight), DWDP_SHAPE="r1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={n}", "--master-addr=127.0.0.1",
                        f"--master-port={29650 + 3 * engine + weight}", os.path.join(ROOT, "tests", "mp_check.py")],
                       env=env, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "failures=0" in out, out[-4000:]


def test_dwdp_rank_timeline_independent_of_a_slow_peer(tmp_path):
    """The paper's no-synchronisation claim on hardware (reference
    tests/test_simcore.cpp:276-311, acceptance criterion 6): the last rank's
    batch doubles; rank 0's DWDP step moves by at most a few percent (only
    shared-link / HBM contention couples the ranks) while its DEP step
    stretches to the slow peer's pace at every all-to-all."""
    import json
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    out = tmp_path / "ind.json"
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", "--master-port=29731",
                        os.path.join(ROOT, "scripts", "independence.py"), "--tokens", "16384",
                        "--layers", "4", "--steps", "4", "--warmup", "2", "--out", str(out)],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    d = json.loads(out.read_text())["rank0"]
    # not slowed by the slow peer (a lighter-loaded link can make rank 0 a
    # few percent faster: the peer pulls its share of rank 0's experts over a
    # longer step, so less HBM / NVLink contention; -5.3% was seen once)
    assert -10.0 < d["dwdp"]["rank0_step_change_pct"] < 5.0, d["dwdp"]
    assert d["dep"]["rank0_step_change_pct"] > 25.0, d["dep"]
