# GEMM2 (and router) on CTA pairs with GEMM1 on the 1-SM kernel (DWDP_GEMM_PAIR=3)
# vs the default all-1-SM build: GPU suite under the variant, then alternating bf16 N=1 benches.
mkdir -p gpurun_out
DWDP_GEMM_PAIR=3 timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/p3_tests.log 2>&1; echo "tests(pair3) rc=$?"; tail -1 gpurun_out/p3_tests.log
for rep in 1 2; do
  for v in 0 3; do
    DWDP_GEMM_PAIR=$v timeout 400 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | grep metric > gpurun_out/p3_${v}_$rep.json
    python -c "import json; d=json.load(open('gpurun_out/p3_${v}_$rep.json')); k=d['kernel_ms_per_layer']; print('pair=$v rep $rep', round(d['value']), {x: round(k[x],3) for x in ('router','permute','gemm1','gemm2','combine','moe')}, d['clocks']['sm_mhz'])"
  done
done
