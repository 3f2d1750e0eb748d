#!/bin/bash
# Round 2: shared-memory carveout on the small layer-path kernels (all vs pull-only), same box, N=1.
mkdir -p gpurun_out
: > gpurun_out/r2_ab_carveout.jsonl
for i in 1 2; do
  for m in all pull; do
    DWDP_CARVEOUT=$m timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-check > gpurun_out/abc_$m.json 2>/dev/null
    python - "$m" <<'PY' >> gpurun_out/r2_ab_carveout.jsonl
import json, sys
d = json.loads(open(f"gpurun_out/abc_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print(json.dumps({"DWDP_CARVEOUT": sys.argv[1], "value": d["value"], "kernel_ms_per_layer": d["kernel_ms_per_layer"],
                  "sm_mhz": d["clocks"]["sm_mhz"]}))
PY
  done
done
cat gpurun_out/r2_ab_carveout.jsonl
