#!/bin/bash
# Round 2: per-kernel times of the router variants (ncu launch list, cold, serialised).
mkdir -p gpurun_out
for m in planes fused; do
  DWDP_ROUTER=$m timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"router|topk|grouped_gemm_kernel|combine" -c 40 --csv --log-file gpurun_out/r2_router_ncu_$m.csv \
    python bench.py --profile --steps 1 --warmup 3 --no-check --no-cpu-baseline --no-e2e > /dev/null 2>&1
  echo "$m rc=$?"
done
