# NVFP4 after the converged-warp MMA issuer + reciprocal quantiser: parity, N=1 benches (nvfp4, fp8), launch list.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nvfp4.py tests/test_gpu.py -q -x -k "fp4 or fp8 or gemm" > gpurun_out/fp4_t2.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/fp4_t2.log
for dt in nvfp4 fp8; do
timeout 600 python bench.py --dtype $dt --no-cpu-baseline > gpurun_out/b1_$dt.log 2>&1; echo "$dt rc=$?"; grep metric gpurun_out/b1_$dt.log > gpurun_out/b1_$dt.json; python -c "import json; d=json.load(open('gpurun_out/b1_$dt.json')); k=d['kernel_ms_per_layer']; print(round(d['value']), round(d['e2e']['value']), {x: round(k[x],2) for x in ('router','permute','gemm1','gemm2','combine','moe')}, round(d['roofline']['achieved']), round(d['roofline']['frac'],3), round(d['roofline']['gemm2_tflops']), d['clocks'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_fp4.csv python bench.py --dtype nvfp4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_fp4.log 2>&1; echo "ncu rc=$?"
