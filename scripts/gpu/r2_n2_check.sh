#!/bin/bash
# Round 2, N=2: multi-GPU suite, then MNT 32K CV 0.2 with the pull engine,
# the auto choice and the MLA window; DWDP + both DEP baselines.
mkdir -p gpurun_out
# (suite ran in r2_multigpu_pytest_n2b.log)

run() {  # name, extra args
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 \
    --master-port=$((29850 + RANDOM % 100)) bench.py --gpus 2 --steps 6 --warmup 3 --no-e2e --tokens 32768 $2 \
    > gpurun_out/r2_bench_n2_32k_$1.json 2> gpurun_out/r2_bench_n2_32k_$1.err
  echo "$1 rc=$?"
}
run pull "--engine pull"
run auto ""
run attn "--attention"
