# NVFP4 CTA-pair GEMM (DWDP_FP4_PAIR=1): GEMM parity first (short timeouts), then layer parity and A/B benches.
mkdir -p gpurun_out
DWDP_FP4_PAIR=1 timeout 240 python -m pytest tests/test_gpu_nvfp4.py -q -x -k "gemm" > gpurun_out/p4_gemm.log 2>&1; echo "gemm rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/p4_gemm.log | head -8
DWDP_FP4_PAIR=1 timeout 400 python -m pytest tests/test_gpu_nvfp4.py -q -x > gpurun_out/p4_all.log 2>&1; echo "all rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/p4_all.log | head -8
for v in 1 0 1; do
DWDP_FP4_PAIR=$v timeout 600 python bench.py --dtype nvfp4 --no-cpu-baseline --no-e2e > gpurun_out/p4_b$v.log 2>&1; echo "pair=$v rc=$?"; grep metric gpurun_out/p4_b$v.log > gpurun_out/p4_b$v.json; python -c "import json; d=json.load(open('gpurun_out/p4_b$v.json')); k=d['kernel_ms_per_layer']; print(round(d['value']), {x: round(k[x],2) for x in ('router','permute','gemm1','gemm2','combine','moe')}, round(d['roofline']['achieved']), round(d['roofline']['gemm2_tflops']), d['clocks']['sm_mhz'])"
done
