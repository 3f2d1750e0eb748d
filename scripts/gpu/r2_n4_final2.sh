#!/bin/bash
# Round 2, N=4 bf16 at HEAD: MNT 64K (default) and 32K, DWDP against all three
# DEPs, per-rank breakdown and the independent-rank rate.
mkdir -p gpurun_out
for tk in 65536 32768; do
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 \
    --master-port=29751 bench.py --gpus 4 --steps 6 --warmup 3 --no-e2e --tokens $tk \
    > gpurun_out/r2_bench_n4_head_$tk.json 2> gpurun_out/r2_bench_n4_head_$tk.err
  echo "bench $tk rc=$?"
  python - $tk <<'PY'
import json, sys
d = json.loads([l for l in open(f"gpurun_out/r2_bench_n4_head_{sys.argv[1]}.json").read().splitlines() if l.startswith("{")][-1])
dep = d["dep_baseline"]
best = max(dep["value"], dep["dedupe"]["value"], dep["dedupe_owners"]["value"])
print(sys.argv[1], "dwdp", round(d["value"]), "indep", round(d["value_independent_ranks"]), "dep0", round(dep["value"]),
      "dep1", round(dep["dedupe"]["value"]), "dep2", round(dep["dedupe_owners"]["value"]),
      "ratio", round(d["value"] / best, 3), "indep ratio", round(d["value_independent_ranks"] / best, 3),
      "exposed", [round(r["gate_wait_ms_per_layer"], 2) for r in d["per_rank"]], d["config"]["prefetch_engine"][0])
PY
done
