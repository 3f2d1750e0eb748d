# Scale prefetch in the scaled epilogues + linear->atom block-scale relayout: full GPU suite, benches, launch list.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/t5.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t5.log
for dt in nvfp4 fp8; do
timeout 600 python bench.py --dtype $dt --no-cpu-baseline > gpurun_out/b1_$dt.log 2>&1; echo "$dt rc=$?"; grep metric gpurun_out/b1_$dt.log > gpurun_out/b1_$dt.json; python -c "import json; d=json.load(open('gpurun_out/b1_$dt.json')); k=d['kernel_ms_per_layer']; print(round(d['value']), round(d['e2e']['value']), {x: round(k[x],2) for x in ('router','permute','gemm1','gemm2','combine','moe')}, round(d['roofline']['achieved']), round(d['roofline']['frac'],3), round(d['roofline']['gemm2_tflops']), d['clocks'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_fp4.csv python bench.py --dtype nvfp4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_fp4.log 2>&1; echo "ncu rc=$?"
