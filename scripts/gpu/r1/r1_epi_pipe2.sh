# Scales of tile i+1 fetched during tile i (double-buffered smem): fp8/fp4 GPU tests + N=1 benches.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu.py tests/test_gpu_nvfp4.py -q -x -k "fp8 or fp4 or pair" > gpurun_out/t7.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t7.log
for dt in nvfp4 fp8; do
timeout 600 python bench.py --dtype $dt --no-cpu-baseline > gpurun_out/b1_$dt.log 2>&1; echo "$dt rc=$?"; grep metric gpurun_out/b1_$dt.log > gpurun_out/b1_$dt.json; python -c "import json; d=json.load(open('gpurun_out/b1_$dt.json')); k=d['kernel_ms_per_layer']; print(round(d['value']), round(d['e2e']['value']), {x: round(k[x],2) for x in ('router','permute','gemm1','gemm2','combine','moe')}, round(d['roofline']['achieved']), round(d['roofline']['frac'],3), round(d['roofline']['gemm2_tflops']), d['clocks'])"
done
