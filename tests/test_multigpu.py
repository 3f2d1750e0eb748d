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
