#!/bin/bash
# Round 2, N=4, MNT 32K bf16: hybrid engine (copy engines + pull kernel on alternating slices) with 37/74/148 pull CTAs
# in flight (DEP off) -- in-step GB/s, exposed time, step throughput.
mkdir -p gpurun_out
: > gpurun_out/r2_hybrid_sweep.jsonl
for ce in 37 74 148; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 \
    --master-port=$((29790 + ce % 97)) bench.py --gpus 4 --steps 6 --warmup 3 --no-e2e --no-dep --tokens 32768 \
    --engine hybrid --pull-ctas $ce > gpurun_out/ce_$ce.json 2> gpurun_out/ce_$ce.err
  echo "ce=$ce rc=$?"
  python - $ce <<'PY' >> gpurun_out/r2_hybrid_sweep.jsonl
import json, sys
ce = sys.argv[1]
d = json.loads([l for l in open(f"gpurun_out/ce_{ce}.json").read().splitlines() if l.startswith("{")][-1])
print(json.dumps({"pull_ctas": int(ce), "value": d["value"], "prefetch_gbs": d["prefetch"]["gbs"],
                  "exposed_ms_per_layer": d["exposed_prefetch_ms_per_layer"],
                  "per_rank_gate_wait": [r["gate_wait_ms_per_layer"] for r in d["per_rank"]],
                  "per_rank_gbs": [r["prefetch_gbs"] for r in d["per_rank"]], "sm_mhz": d["clocks"]["sm_mhz"]}))
PY
done
cat gpurun_out/r2_hybrid_sweep.jsonl
