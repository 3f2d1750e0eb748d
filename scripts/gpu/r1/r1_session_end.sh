# Session-end check of HEAD: GPU suite, smoke, default N=1 bench, and the launch list
# (gpu__time_duration per launch, one 1-layer step) for kernel shares.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/se_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/se_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 400 python bench.py > gpurun_out/se_b1.log 2>&1; echo "bench rc=$?"; grep metric gpurun_out/se_b1.log > gpurun_out/se_b1.json
python -c "import json; d=json.load(open('gpurun_out/se_b1.json')); k=d['kernel_ms_per_layer']; print(round(d['value']), round(d['e2e']['value']), {x: round(k[x],3) for x in ('router','permute','gemm1','gemm2','combine','moe')}, round(d['roofline']['frac'],3), d['clocks'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/se_launches.csv python bench.py --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/se_ncu.log 2>&1; echo "ncu rc=$?"
