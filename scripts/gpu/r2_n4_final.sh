#!/bin/bash
# Round 2, N=4 after the co-residency fixes: MNT 64K (default), MNT 32K auto,
# MNT 32K with the sm_100a MLA block in the window; DWDP + both DEP baselines.
mkdir -p gpurun_out
run() {  # name, extra args
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 \
    --master-port=$((29850 + RANDOM % 100)) bench.py --gpus 4 --steps 6 --warmup 3 --no-e2e $2 \
    > gpurun_out/r2_bench_n4_$1.json 2> gpurun_out/r2_bench_n4_$1.err
  echo "$1 rc=$?"
}
run mnt64k ""
run mnt32k "--tokens 32768"
run mnt32k_attn "--tokens 32768 --attention"
