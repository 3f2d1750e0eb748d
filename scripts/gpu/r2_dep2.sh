#!/bin/bash
# Round 2, N=2: multi-GPU parity incl. DEP mode 1 and the independence test,
# then the default bench at N=2 (DWDP + both DEP baselines on the same box).
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_multigpu.py -q -x -p no:cacheprovider > gpurun_out/r2_multigpu_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_multigpu_pytest.log
tail -3 gpurun_out/r2_multigpu_pytest.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 \
  --master-port=29721 bench.py --gpus 2 --steps 6 --warmup 3 --no-e2e > gpurun_out/r2_bench_n2.json 2> gpurun_out/r2_bench_n2.err
echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads([l for l in open("gpurun_out/r2_bench_n2.json").read().splitlines() if l.startswith("{")][-1])
dep = d["dep_baseline"]
print(json.dumps({"dwdp": d["value"], "exposed": d["exposed_prefetch_ms_per_layer"], "dep": dep["value"],
                  "dwdp_over_dep": dep["dwdp_over_dep"], "dep_comm": dep["comm_ms_per_layer"],
                  "dedupe": {k: dep["dedupe"][k] for k in ("value", "dwdp_over_dep", "comm_ms_per_layer")} if dep.get("dedupe") else None,
                  "clocks": d["clocks"]}))
PY
