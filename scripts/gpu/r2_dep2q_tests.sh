#!/bin/bash
# Round 2, N=2: multi-GPU parity after DEP mode 1 for quantised experts.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -k "match_all_local" > gpurun_out/r2_dep2q_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_dep2q_pytest.log
tail -3 gpurun_out/r2_dep2q_pytest.log
grep -h "DEP mode 1\|MPCHECK" gpurun_out/r2_dep2q_pytest.log | head
