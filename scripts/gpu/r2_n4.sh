#!/bin/bash
# Round 2, N=4: default bench (MNT 64K) and MNT 32K, CV 0.2, DWDP + both DEP baselines.
mkdir -p gpurun_out
for mnt in 65536 32768; do
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 \
    --master-port=$((29800 + mnt % 97)) bench.py --gpus 4 --steps 6 --warmup 3 --no-e2e --tokens $mnt \
    > gpurun_out/r2_bench_n4_mnt$mnt.json 2> gpurun_out/r2_bench_n4_mnt$mnt.err
  echo "bench mnt=$mnt rc=$?"
done
timeout 900 python -m pytest tests/test_multigpu.py -q -x -p no:cacheprovider -k "r1_shapes or dedupe or match_all_local" > gpurun_out/r2_multigpu_pytest_n4.log 2>&1
echo "pytest n4 rc=$?"; tail -2 gpurun_out/r2_multigpu_pytest_n4.log
