# bf16 A/B, alternating on one box: 1-SM GEMMs (default) vs CTA pairs for GEMM1 only (DWDP_GEMM_PAIR=2).
mkdir -p gpurun_out
DWDP_GEMM_PAIR=2 timeout 300 python -m pytest tests/test_gpu.py -q -x -k "moe_forward or pair" > gpurun_out/ab1_t.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/ab1_t.log
for v in 0 2 0 2; do
DWDP_GEMM_PAIR=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab1_$v.log 2>&1; grep metric gpurun_out/ab1_$v.log > gpurun_out/ab1_$v.json; python -c "import json; d=json.load(open('gpurun_out/ab1_$v.json')); k=d['kernel_ms_per_layer']; print('pair=$v', round(d['value']), {x: round(k[x],2) for x in ('router','permute','gemm1','gemm2','combine','moe')}, d['clocks']['sm_mhz'])"
done
