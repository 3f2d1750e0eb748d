# Software-pipelined TMEM loads in the plain (GEMM2) epilogue: full GPU suite + N=1 benches of all three dtypes.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/t6.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t6.log
for dt in nvfp4 fp8 bf16; do
timeout 600 python bench.py --dtype $dt --no-cpu-baseline > gpurun_out/b1_$dt.log 2>&1; echo "$dt rc=$?"; grep metric gpurun_out/b1_$dt.log > gpurun_out/b1_$dt.json; python -c "import json; d=json.load(open('gpurun_out/b1_$dt.json')); k=d['kernel_ms_per_layer']; print(round(d['value']), round(d['e2e']['value']), {x: round(k[x],2) for x in ('router','permute','gemm1','gemm2','combine','moe')}, round(d['roofline']['achieved']), round(d['roofline']['frac'],3), round(d['roofline']['gemm2_tflops']), d['clocks'])"
done
