# Round-end check of HEAD: full GPU suite, smoke, default bench and the NVFP4 bench (N=1).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/fc4_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/fc4_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/fc4_b1.json 2> gpurun_out/fc4_b1.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('gpurun_out/fc4_b1.json')); k=d['kernel_ms_per_layer']; print(round(d['value']), round(d['e2e']['value']), {x: round(k[x],2) for x in ('gemm1','gemm2','moe')}, round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
timeout 600 python bench.py --dtype nvfp4 --no-cpu-baseline > gpurun_out/fc4_b4.log 2>&1; grep metric gpurun_out/fc4_b4.log > gpurun_out/fc4_b4.json; python -c "import json; d=json.load(open('gpurun_out/fc4_b4.json')); k=d['kernel_ms_per_layer']; print(round(d['value']), round(d['e2e']['value']), {x: round(k[x],2) for x in ('router','permute','gemm1','gemm2','combine','moe')}, round(d['roofline']['achieved']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
