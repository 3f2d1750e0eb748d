# NVFP4 GEMM2 on CTA pairs (DWDP_FP4_PAIR2=1) vs 1-SM after the drain-order change: same-box A/B.
mkdir -p gpurun_out
for v in 0 1 0 1; do
DWDP_FP4_PAIR2=$v timeout 600 python bench.py --dtype nvfp4 --no-cpu-baseline --no-e2e > gpurun_out/pb.log 2>&1; grep metric gpurun_out/pb.log > gpurun_out/pb$v.json; python -c "import json; d=json.load(open('gpurun_out/pb$v.json')); k=d['kernel_ms_per_layer']; print('pair2=$v', round(d['value']), {x: round(k[x],2) for x in ('gemm1','gemm2','moe')}, d['clocks']['sm_mhz'])"
done
