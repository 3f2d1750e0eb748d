#!/bin/bash
# Round 2: correctness of the fixed skip-ahead + split layout, then a same-box
# A/B of the default N=1 bench: DWDP_GEMM_PAIR unset (all 1-SM) vs =4 (split
# layout: GEMM1 1-SM on 128-row segments, GEMM2 on CTA pairs), alternating.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_runtime.py tests/test_gpu.py -q -x -p no:cacheprovider -k "runtime or pair or skip" > gpurun_out/r2_split_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_split_pytest.log
tail -3 gpurun_out/r2_split_pytest.log
: > gpurun_out/r2_ab_split.jsonl
for i in 1 2; do
  for m in 0 4; do
    DWDP_GEMM_PAIR=$m timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_$m.json 2>/dev/null
    python - "$m" <<'PY' >> gpurun_out/r2_ab_split.jsonl
import json, sys
d = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print(json.dumps({"DWDP_GEMM_PAIR": sys.argv[1], "value": d["value"], "kernel_ms_per_layer": d["kernel_ms_per_layer"],
                  "sm_mhz": d["clocks"]["sm_mhz"], "reasons": d["clocks"]["reasons"]}))
PY
  done
done
cat gpurun_out/r2_ab_split.jsonl
