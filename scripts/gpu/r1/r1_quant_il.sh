# Lane-interleaved NVFP4 row quantiser for H: bit-exact tests + bench.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_nvfp4.py -q -x > gpurun_out/qil_t.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/qil_t.log | head -5
for i in 1 2; do
timeout 600 python bench.py --dtype nvfp4 --no-cpu-baseline > gpurun_out/qil_b.log 2>&1; grep metric gpurun_out/qil_b.log > gpurun_out/qil_b$i.json; python -c "import json; d=json.load(open('gpurun_out/qil_b$i.json')); k=d['kernel_ms_per_layer']; print(round(d['value']), round(d['e2e']['value']), {x: round(k[x],2) for x in ('router','permute','gemm1','gemm2','combine','moe')}, d['clocks']['sm_mhz'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --kernel-name regex:"quant_rows" -c 2 --csv --log-file gpurun_out/qil_ncu.csv python bench.py --dtype nvfp4 --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"; grep -E "duration|dram" gpurun_out/qil_ncu.csv | cut -d, -f5,13- | head
