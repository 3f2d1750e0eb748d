#!/bin/bash
# Round 2, N=2: config-4 CV x MNT sweep (fp8) at HEAD, DWDP against all three DEPs.
mkdir -p gpurun_out
for dt in fp8; do
  rm -f gpurun_out/r2_sweep_n2_$dt.jsonl
  timeout 2400 python scripts/sweep.py --gpus 2 --cv 0,0.1,0.2,0.3 --tokens 32768,65536 --steps 4 --warmup 3 \
    --extra "--dtype $dt" --out gpurun_out/r2_sweep_n2_$dt.jsonl
  echo "sweep $dt rc=$?"
  python - $dt <<'PY'
import json, sys
for l in open(f"gpurun_out/r2_sweep_n2_{sys.argv[1]}.jsonl"):
    d = json.loads(l)
    if "error" in d:
        print(d["mnt"], d["cv"], "ERROR", d["error"][-300:]); continue
    print(sys.argv[1], d["mnt"], d["cv"], round(d["dwdp_tokens_per_s_per_gpu"]), round(d["dep_tokens_per_s_per_gpu"]),
          round(d["dep_mode1_tokens_per_s_per_gpu"]), round(d["dep_mode2_tokens_per_s_per_gpu"]),
          "best", round(d["dwdp_over_best_dep"], 3), "exposed", round(d["exposed_prefetch_ms_per_layer"], 2), d["engine"][0])
PY
done
