# Plain epilogue: overlapped chunks read and released first, 3-deep TMEM load pipeline. Full GPU suite + benches.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/e3_t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/e3_t.log
for dt in nvfp4 nvfp4 bf16 fp8; do
timeout 600 python bench.py --dtype $dt --no-cpu-baseline --no-e2e > gpurun_out/e3_b.log 2>&1; grep metric gpurun_out/e3_b.log > gpurun_out/e3_$dt.json; python -c "import json; d=json.load(open('gpurun_out/e3_$dt.json')); k=d['kernel_ms_per_layer']; print('$dt', round(d['value']), {x: round(k[x],2) for x in ('gemm1','gemm2','moe')}, d['clocks']['sm_mhz'])"
done
