#!/bin/bash
# Round 2, N=4: MNT 32K with the TS-mode MLA block in the prefetch window,
# DWDP against all three DEPs (the attention runs in every arm).
mkdir -p gpurun_out
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 \
  --master-port=29877 bench.py --gpus 4 --steps 6 --warmup 3 --no-e2e --tokens 32768 --attention \
  > gpurun_out/r2_bench_n4_mnt32k_attention2.json 2> gpurun_out/r2_bench_n4_mnt32k_attention2.err
echo "rc=$?"; tail -2 gpurun_out/r2_bench_n4_mnt32k_attention2.err
python - <<'PY'
import json
d = json.loads([l for l in open("gpurun_out/r2_bench_n4_mnt32k_attention2.json").read().splitlines() if l.startswith("{")][-1])
dep = d["dep_baseline"]
print("dwdp", round(d["value"]), "dep0", round(dep["value"]), "dep1", round(dep["dedupe"]["value"]),
      "dep2", round(dep["dedupe_owners"]["value"]), "best", round(dep["dwdp_over_best_dep"], 3),
      "exposed", round(d["exposed_prefetch_ms_per_layer"], 3), "attention", json.dumps(d.get("attention"))[:300])
PY
