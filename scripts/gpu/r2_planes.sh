#!/bin/bash
# Round 2: router planes emitted by the previous layer's combine -- parity
# (stack vs layer-by-layer bitwise, routing, headline), N=1 bench, launch list.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_headline.py -q -x -p no:cacheprovider > gpurun_out/r2_planes_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_planes_pytest.log
tail -3 gpurun_out/r2_planes_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_planes_bench.json 2> gpurun_out/r2_planes_bench.err
echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2_planes_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], {k: round(v, 3) for k, v in d['kernel_ms_per_layer'].items()}, d['clocks'], d['check']['ok'], d['gpu_launches'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r2_planes_launches.csv python bench.py --steps 2 --warmup 1 --no-check --no-cpu-baseline --no-e2e \
  > gpurun_out/r2_planes_ncu.log 2>&1
echo "ncu rc=$?"
python scripts/launch_shares.py gpurun_out/r2_planes_launches.csv gpurun_out/r2_planes_launches_summary.json | tail -12
