# Round-end check of HEAD: full GPU suite, smoke, default bench (N=1), reference arm.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/fc3_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/fc3_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/fc3_b1.json 2> gpurun_out/fc3_b1.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('gpurun_out/fc3_b1.json')); k=d['kernel_ms_per_layer']; print(round(d['value']), round(d['e2e']['value']), {x: round(k[x],2) for x in ('gemm1','gemm2','moe')}, round(d['roofline']['frac'],3), d['roofline']['traffic'], d['cpu_baseline']['value'], d['gpu_launches'], d['clocks'])"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fc3_ref.json 2>&1; echo "ref rc=$?"; tail -c 300 gpurun_out/fc3_ref.json
