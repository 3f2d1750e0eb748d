#!/bin/bash
# Round 2, N=4 MNT 32K + attention: two-tile kernel vs one-tile kernel, same box, per rank.
mkdir -p gpurun_out
for v in 1 0 1; do
  DWDP_ATTN_PAIR=$v timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 \
    --master-port=$((29880 + v)) bench.py --gpus 4 --steps 6 --warmup 3 --no-e2e --tokens 32768 --attention --no-dep \
    > gpurun_out/r2_n4_attn5_$v.json 2> gpurun_out/r2_n4_attn5_$v.err
  echo "pair=$v rc=$?"
  python - $v <<'PY'
import json, sys
d = json.loads([l for l in open(f"gpurun_out/r2_n4_attn5_{sys.argv[1]}.json").read().splitlines() if l.startswith("{")][-1])
print("pair", sys.argv[1], "dwdp", round(d["value"]), [(r["rank"], round(r["ms_per_step"], 1), round(r["attention_ms_per_layer"], 2), round(r["moe_ms_per_layer"], 2)) for r in d["per_rank"]])
PY
done
