#!/bin/bash
# Round 2, N=4: DWDP independence (rank 3's batch x2; rank 0's timeline) vs DEP.
mkdir -p gpurun_out
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 \
  --master-port=29961 scripts/independence.py --out gpurun_out/r2_independence_n4.json \
  > gpurun_out/r2_independence_n4.log 2>&1
echo "independence rc=$?"
tail -c 1500 gpurun_out/r2_independence_n4.log
