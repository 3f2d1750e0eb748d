#!/bin/bash
# Round 2, N=4: DEP modes 1 and 2 with fp8 / nvfp4 experts (quantised rows on the wire) -- multi-GPU parity
# (mp_check: DWDP, DEP mode 0 bit-identical, mode 1 within 1e-2 of all-local),
# then DWDP vs both DEP baselines at MNT 32K and 64K in fp8 and nvfp4.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -k "match_all_local" > gpurun_out/r2_qwire_n4_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_qwire_n4_pytest.log
tail -3 gpurun_out/r2_qwire_n4_pytest.log
for dt in fp8 nvfp4; do
  for tk in 32768 65536; do
    timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 \
      --master-port=29731 bench.py --gpus 4 --steps 6 --warmup 3 --no-e2e --dtype $dt --tokens $tk \
      > gpurun_out/r2_bench_n4_${dt}_${tk}_qwire.json 2> gpurun_out/r2_bench_n4_${dt}_${tk}_qwire.err
    echo "bench $dt $tk rc=$?"
    python - "$dt" "$tk" <<'PY'
import json, sys
dt, tk = sys.argv[1], sys.argv[2]
d = json.loads([l for l in open(f"gpurun_out/r2_bench_n4_{dt}_{tk}_qwire.json").read().splitlines() if l.startswith("{")][-1])
dep = d["dep_baseline"]; q = dep.get("dedupe") or {}
q2 = dep.get("dedupe_owners") or {}
print(dt, tk, "dwdp", round(d["value"]), "dep0", round(dep["value"]), "dep1", round(q.get("value", 0)),
      "dep2", round(q2.get("value", 0)), "best", round(dep.get("dwdp_over_best_dep", 0), 3),
      "exposed", round(d["exposed_prefetch_ms_per_layer"], 3))
PY
  done
done
