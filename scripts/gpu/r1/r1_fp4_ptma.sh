# NVFP4 CTA-pair kernel with TMA-store epilogues (4 stages): parity, then A/B of GEMM2 on pairs (DWDP_FP4_PAIR2).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_nvfp4.py -q -x > gpurun_out/pt_t.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/pt_t.log | head -8
DWDP_FP4_PAIR2=1 timeout 600 python -m pytest tests/test_gpu_nvfp4.py -q -x -k "moe_forward or dwdp" > gpurun_out/pt_t2.log 2>&1; echo "tests pair2 rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/pt_t2.log | head -8
for v in 0 1 0 1; do
DWDP_FP4_PAIR2=$v timeout 600 python bench.py --dtype nvfp4 --no-cpu-baseline --no-e2e > gpurun_out/pt_b.log 2>&1; grep metric gpurun_out/pt_b.log > gpurun_out/pt_b$v.json; python -c "import json; d=json.load(open('gpurun_out/pt_b$v.json')); k=d['kernel_ms_per_layer']; print('pair2=$v', round(d['value']), {x: round(k[x],2) for x in ('gemm1','gemm2','moe')}, d['clocks']['sm_mhz'])"
done
