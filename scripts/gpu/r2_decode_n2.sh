#!/bin/bash
# Round 2, N=2: config-5 decode sweep (fp8, split fetch, Zipf 0 / 1.2) against all three DEPs.
mkdir -p gpurun_out
rm -f gpurun_out/r2_sweep_decode_n2.jsonl
timeout 2700 python scripts/sweep_decode.py --gpus 2 --batch 64,256,1024,4096 --zipf 0,1.2 --fetch split \
  --out gpurun_out/r2_sweep_decode_n2.jsonl > /dev/null 2>&1
echo "sweep rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/r2_sweep_decode_n2.jsonl"):
    d = json.loads(l)
    if "error" in d:
        print(d.get("batch"), d.get("zipf"), "ERROR", d["error"][-200:]); continue
    print(d["batch"], d["zipf"], "dwdp ms", round(d["dwdp_ms_per_step"], 1), "dep ms", round(d["dep_ms_per_step"], 1),
          round(d["dep_mode1_ms_per_step"] or 0, 1), round(d["dep_mode2_ms_per_step"] or 0, 1), "best", round(d["dwdp_over_best_dep"] or 0, 3))
PY
