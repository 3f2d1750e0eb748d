#!/bin/bash
# Round 2, N=2: multi-GPU parity (MID + R1 shapes, DWDP and DEP == all-local)
# and the hardware independence experiment (scripts/independence.py).
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/r2_topo.txt 2>&1
timeout 1500 python -m pytest tests/test_multigpu.py -q -x -p no:cacheprovider > gpurun_out/r2_multigpu_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_multigpu_pytest.log
tail -3 gpurun_out/r2_multigpu_pytest.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 \
  --master-port=29711 scripts/independence.py --out gpurun_out/r2_independence_n2.json \
  > gpurun_out/r2_independence_n2.log 2>&1
echo "independence rc=$?"
tail -c 1500 gpurun_out/r2_independence_n2.log
