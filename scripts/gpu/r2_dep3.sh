#!/bin/bash
# Round 2: DEP mode 2 (owner-only dispatch) -- multi-GPU parity, then the
# default bench (bf16, MNT 64K) and MNT 32K with all three DEP baselines.
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 2400 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -k "match_all_local" > gpurun_out/r2_dep3_n${NG}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_dep3_n${NG}_pytest.log
tail -3 gpurun_out/r2_dep3_n${NG}_pytest.log
grep -h "DEP mode" gpurun_out/r2_dep3_n${NG}_pytest.log | head -5
for tk in 65536 32768; do
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr=127.0.0.1 \
    --master-port=29741 bench.py --gpus $NG --steps 6 --warmup 3 --no-e2e --tokens $tk \
    > gpurun_out/r2_bench_n${NG}_dep3_${tk}.json 2> gpurun_out/r2_bench_n${NG}_dep3_${tk}.err
  echo "bench $tk rc=$?"; tail -2 gpurun_out/r2_bench_n${NG}_dep3_${tk}.err
  python - "$NG" "$tk" <<'PY'
import json, sys
ng, tk = sys.argv[1], sys.argv[2]
d = json.loads([l for l in open(f"gpurun_out/r2_bench_n{ng}_dep3_{tk}.json").read().splitlines() if l.startswith("{")][-1])
dep = d["dep_baseline"]
print(ng, tk, "dwdp", round(d["value"]), "dep0", round(dep["value"]), "dep1", round(dep["dedupe"]["value"]),
      "dep2", round(dep["dedupe_owners"]["value"]), "best ratio", round(dep["dwdp_over_best_dep"], 3),
      "comm ms/layer", round(dep["comm_ms_per_layer"], 2), round(dep["dedupe"]["comm_ms_per_layer"], 2),
      round(dep["dedupe_owners"]["comm_ms_per_layer"], 2), "exposed", round(d["exposed_prefetch_ms_per_layer"], 3))
PY
done
