#!/bin/bash
# Round 2: router GEMM on CTA pairs (DWDP_ROUTER_PAIR=1) vs the 1-SM kernel --
# routing parity with the pair router, ncu launch times, step A/B on one box.
mkdir -p gpurun_out
DWDP_ROUTER_PAIR=1 timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_headline.py -q -x -p no:cacheprovider -k "route or moe_forward or headline or stack" > gpurun_out/r2_router_pair_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_router_pair_pytest.log
tail -3 gpurun_out/r2_router_pair_pytest.log
for P in 1 0; do
  DWDP_ROUTER_PAIR=$P timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"router_gemm" -c 10 --csv --log-file gpurun_out/r2_router_pair_ncu_$P.csv \
    python bench.py --profile --steps 1 --warmup 3 --no-check --no-cpu-baseline --no-e2e > /dev/null 2>&1
  echo "pair=$P ncu rc=$?"; grep router_gemm gpurun_out/r2_router_pair_ncu_$P.csv | awk -F'","' '{print $NF}' | head -4 | tr '\n' ' '; echo
done
for P in 1 0 1 0; do
  DWDP_ROUTER_PAIR=$P timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/rp_$P.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/rp_$P.json').read().strip().splitlines()[-1])
print('pair=$P', round(d['value']), {k: round(v, 3) for k, v in d['kernel_ms_per_layer'].items() if k in ('router', 'gemm1', 'gemm2')}, d['clocks']['sm_mhz'], d['check']['ok'])"
done
