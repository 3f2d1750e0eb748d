#!/bin/bash
# Round 2, N=4, MNT 32K CV 0.2: engine choice (auto probe logged, forced pull)
# and the paper's window with the sm_100a MLA block (--attention).
mkdir -p gpurun_out
run() {  # name, extra args
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 \
    --master-port=$((29850 + RANDOM % 100)) bench.py --gpus 4 --steps 6 --warmup 3 --no-e2e --tokens 32768 $2 \
    > gpurun_out/r2_bench_n4_32k_$1.json 2> gpurun_out/r2_bench_n4_32k_$1.err
  echo "$1 rc=$?"
}
run auto ""
run pull "--engine pull"
run attn "--attention"
