#!/bin/bash
# Round 2, N=4: MNT 32K with the two-tile MLA block (default) in the window, per-rank
# breakdown (auto engine, then the pull engine forced).
mkdir -p gpurun_out
for eng in auto; do
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 \
    --master-port=29878 bench.py --gpus 4 --steps 6 --warmup 3 --no-e2e --tokens 32768 --attention --engine $eng \
    > gpurun_out/r2_bench_n4_mnt32k_attention4_$eng.json 2> gpurun_out/r2_bench_n4_mnt32k_attention4_$eng.err
  echo "$eng rc=$?"; tail -1 gpurun_out/r2_bench_n4_mnt32k_attention4_$eng.err
  python - $eng <<'PY'
import json, sys
d = json.loads([l for l in open(f"gpurun_out/r2_bench_n4_mnt32k_attention4_{sys.argv[1]}.json").read().splitlines() if l.startswith("{")][-1])
dep = d["dep_baseline"]
print("dwdp", round(d["value"]), "dep0", round(dep["value"]), "dep1", round(dep["dedupe"]["value"]),
      "dep2", round(dep["dedupe_owners"]["value"]), "best", round(dep["dwdp_over_best_dep"], 3), d["config"]["prefetch_engine"][0])
for r in d["per_rank"]:
    print({k: (round(v, 2) if isinstance(v, float) else v) for k, v in r.items()})
PY
done
