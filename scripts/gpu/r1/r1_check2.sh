# Full GPU suite + smoke + default bench; fp8 A/B of GEMM1 on CTA pairs (DWDP_GEMM_PAIR=2).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/c2_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c2_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/c2_b1.json 2> gpurun_out/c2_b1.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('gpurun_out/c2_b1.json')); k=d['kernel_ms_per_layer']; print(round(d['value']), round(d['e2e']['value']), {x: round(k[x],2) for x in ('gemm1','gemm2','moe')}, round(d['roofline']['frac'],3), d['cpu_baseline']['value'], d['clocks']['sm_mhz'])"
for v in 0 2; do
DWDP_GEMM_PAIR=$v timeout 600 python bench.py --dtype fp8 --no-cpu-baseline --no-e2e > gpurun_out/c2_f8_$v.log 2>&1; grep metric gpurun_out/c2_f8_$v.log > gpurun_out/c2_f8_$v.json; python -c "import json; d=json.load(open('gpurun_out/c2_f8_$v.json')); k=d['kernel_ms_per_layer']; print('fp8 pair=$v', round(d['value']), {x: round(k[x],2) for x in ('gemm1','gemm2','moe')}, d['clocks']['sm_mhz'])"
done
