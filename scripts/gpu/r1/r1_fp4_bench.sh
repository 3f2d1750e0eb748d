# NVFP4 path: parity tests, N=1 bench (config-2 shapes), launch list and a full ncu capture of the FP4 GEMMs.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_nvfp4.py -q > gpurun_out/fp4_all.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/fp4_all.log
timeout 600 python bench.py --dtype nvfp4 --no-cpu-baseline > gpurun_out/fp4_b1.log 2>&1; echo "b1 rc=$?"; grep metric gpurun_out/fp4_b1.log > gpurun_out/fp4_b1.json; python -c "import json; d=json.load(open('gpurun_out/fp4_b1.json')); k=d['kernel_ms_per_layer']; print(round(d['value']), round(d['e2e']['value']), {x: round(k[x],2) for x in ('router','permute','gemm1','gemm2','combine','moe')}, round(d['roofline']['achieved']), round(d['roofline']['frac'],3), d['roofline']['gemm2_tflops'], d['clocks'])"
tail -3 gpurun_out/fp4_b1.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"grouped_gemm_kernel" --launch-skip 10 -c 3 -o gpurun_out/fp4_gemm -f python bench.py --dtype nvfp4 --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/fp4_ncu.log 2>&1; echo "ncu rc=$?"
