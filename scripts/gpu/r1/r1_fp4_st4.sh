# NVFP4 1-SM kernel with 4 stages (219 KB smem): parity + N=1 bench.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_nvfp4.py -q -x > gpurun_out/st4_t.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/st4_t.log | head -8
for i in 1 2; do
timeout 600 python bench.py --dtype nvfp4 --no-cpu-baseline --no-e2e > gpurun_out/st4_b.log 2>&1; echo "rc=$?"; grep metric gpurun_out/st4_b.log > gpurun_out/st4_b.json; python -c "import json; d=json.load(open('gpurun_out/st4_b.json')); k=d['kernel_ms_per_layer']; print(round(d['value']), {x: round(k[x],2) for x in ('router','permute','gemm1','gemm2','combine','moe')}, round(d['roofline']['achieved']), round(d['roofline']['gemm2_tflops']), d['clocks']['sm_mhz'])"
done
