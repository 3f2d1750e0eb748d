# NVFP4 1-SM kernel with two epilogue warp groups (12 warps): parity + bench (default config) + A/B of GEMM1 pair off.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_nvfp4.py -q -x > gpurun_out/e8_t.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/e8_t.log | head -8
for v in 1 0; do
DWDP_FP4_PAIR=$v timeout 600 python bench.py --dtype nvfp4 --no-cpu-baseline > gpurun_out/e8_b$v.log 2>&1; echo "pair=$v rc=$?"; grep metric gpurun_out/e8_b$v.log > gpurun_out/e8_b$v.json; python -c "import json; d=json.load(open('gpurun_out/e8_b$v.json')); k=d['kernel_ms_per_layer']; print(round(d['value']), round(d['e2e']['value']), {x: round(k[x],2) for x in ('router','permute','gemm1','gemm2','combine','moe')}, round(d['roofline']['achieved']), round(d['roofline']['gemm2_tflops']), d['clocks']['sm_mhz'])"
done
