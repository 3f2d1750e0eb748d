# fp8 (W8A8) experts, N=1: all-1-SM (default) vs GEMM2-only pairs (=3) vs every GEMM on pairs (=1).
mkdir -p gpurun_out
for rep in 1 2; do
  for v in 0 3 1; do
    DWDP_GEMM_PAIR=$v timeout 400 python bench.py --dtype fp8 --no-cpu-baseline --no-e2e 2>/dev/null | grep metric > gpurun_out/pf8_${v}_$rep.json
    python -c "import json; d=json.load(open('gpurun_out/pf8_${v}_$rep.json')); k=d['kernel_ms_per_layer']; print('fp8 pair=$v rep $rep', round(d['value']), {x: round(k[x],3) for x in ('router','permute','gemm1','gemm2','combine','moe')}, d['clocks']['sm_mhz'])"
  done
done
