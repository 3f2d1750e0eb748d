#!/bin/bash
# Round 2: router GEMM with the three weight planes stacked as one N192 B operand --
# routing parity (bit-exact incl. the headline batch), ncu launch times, step A/B
# is against the previous build's numbers (profiles/r2_router_ncu_fused.csv).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu.py tests/test_gpu_headline.py -q -x -p no:cacheprovider -k "route or moe_forward or headline" > gpurun_out/r2_router_stacked_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_router_stacked_pytest.log
tail -3 gpurun_out/r2_router_stacked_pytest.log
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"router|topk|grouped_gemm_kernel|combine" -c 40 --csv --log-file gpurun_out/r2_router_ncu_stacked.csv \
  python bench.py --profile --steps 1 --warmup 3 --no-check --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "ncu rc=$?"
grep router_gemm gpurun_out/r2_router_ncu_stacked.csv | awk -F'","' '{print $NF}' | head -5
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_router_stacked_bench.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2_router_stacked_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['kernel_ms_per_layer'], d['clocks'])"
