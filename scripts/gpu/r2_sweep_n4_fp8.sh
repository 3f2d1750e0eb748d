#!/bin/bash
# Round 2, N=4: config-4 CV x MNT sweep (fp8 experts) at HEAD, DWDP against all three DEPs.
mkdir -p gpurun_out
rm -f gpurun_out/r2_sweep_n4_fp8.jsonl
timeout 3000 python scripts/sweep.py --gpus 4 --cv 0,0.1,0.2,0.3 --tokens 32768,65536 --steps 4 --warmup 3 --extra "--dtype fp8" \
  --out gpurun_out/r2_sweep_n4_fp8.jsonl
echo "sweep rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/r2_sweep_n4_fp8.jsonl"):
    d = json.loads(l)
    if "error" in d:
        print(d["mnt"], d["cv"], "ERROR", d["error"][-300:]); continue
    print(d["mnt"], d["cv"], round(d["dwdp_tokens_per_s_per_gpu"]), round(d["dep_tokens_per_s_per_gpu"]),
          round(d["dep_mode1_tokens_per_s_per_gpu"]), round(d["dep_mode2_tokens_per_s_per_gpu"]),
          "best", round(d["dwdp_over_best_dep"], 3), "indep/gpu", round(d["dwdp_independent_ranks_per_gpu"] or 0),
          "exposed", round(d["exposed_prefetch_ms_per_layer"], 2), d["engine"][0])
PY
