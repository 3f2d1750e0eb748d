# NVFP4 GEMM2 with the TMA-store epilogue: parity + N=1 bench (twice).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_nvfp4.py -q -x > gpurun_out/ts_t.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/ts_t.log | head -8
for i in 1 2; do
timeout 600 python bench.py --dtype nvfp4 --no-cpu-baseline > gpurun_out/ts_b.log 2>&1; echo "rc=$?"; grep metric gpurun_out/ts_b.log > gpurun_out/ts_b$i.json; python -c "import json; d=json.load(open('gpurun_out/ts_b$i.json')); k=d['kernel_ms_per_layer']; print(round(d['value']), round(d['e2e']['value']), {x: round(k[x],2) for x in ('router','permute','gemm1','gemm2','combine','moe')}, round(d['roofline']['gemm2_tflops']), d['clocks']['sm_mhz'])"
done
