#!/bin/bash
# Round 2: the N=8 code path (7 peers' IPC arenas, 224 pulled experts per
# layer, R1 shapes) emulated as 8 ranks on 4 GPUs (--oversubscribe: numbers
# are not bench values; DEP off), MNT 8192, 2 layers.
mkdir -p gpurun_out
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=8 --master-addr=127.0.0.1 \
  --master-port=29911 bench.py --gpus 8 --steps 3 --warmup 3 --no-e2e --tokens 8192 --layers 2 --oversubscribe \
  > gpurun_out/r2_n8_emul.json 2> gpurun_out/r2_n8_emul.err
echo "n8 emul rc=$?"; tail -c 600 gpurun_out/r2_n8_emul.json
