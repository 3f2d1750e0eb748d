#!/bin/bash
# Round 2: fused router GEMM -- routing parity (bit-exact incl. the headline
# batch), then a same-box A/B against the plane-product router (DWDP_ROUTER=planes).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu.py tests/test_gpu_headline.py -q -x -p no:cacheprovider -k "route or moe_forward or headline or gemm_pair" > gpurun_out/r2_router_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_router_pytest.log
tail -3 gpurun_out/r2_router_pytest.log
: > gpurun_out/r2_ab_router.jsonl
for i in 1 2; do
  for m in planes fused; do
    DWDP_ROUTER=$m timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/abr_$m.json 2>/dev/null
    python - "$m" <<'PY' >> gpurun_out/r2_ab_router.jsonl
import json, sys
d = json.loads(open(f"gpurun_out/abr_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print(json.dumps({"DWDP_ROUTER": sys.argv[1], "value": d["value"], "kernel_ms_per_layer": d["kernel_ms_per_layer"],
                  "sm_mhz": d["clocks"]["sm_mhz"], "reasons": d["clocks"]["reasons"]}))
PY
  done
done
cat gpurun_out/r2_ab_router.jsonl
