# NVFP4: permute batching (parity), raster A/B (auto / m-block-major / n-block-major inside expert segments).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_nvfp4.py -q -x > gpurun_out/ra_t.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/ra_t.log | head -5
for r in auto m n auto; do
if [ $r = auto ]; then unset DWDP_RASTER; else export DWDP_RASTER=$r; fi
timeout 600 python bench.py --dtype nvfp4 --no-cpu-baseline --no-e2e > gpurun_out/ra.log 2>&1; grep metric gpurun_out/ra.log > gpurun_out/ra_$r.json; python -c "import json; d=json.load(open('gpurun_out/ra_$r.json')); k=d['kernel_ms_per_layer']; print('raster=$r', round(d['value']), {x: round(k[x],2) for x in ('permute','gemm1','gemm2','moe')}, d['clocks']['sm_mhz'])"
done
