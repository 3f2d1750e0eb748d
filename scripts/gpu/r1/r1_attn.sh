# MLA attention stand-in in the prefetch window: its test, N=1 bench with --attention.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_attention.py -q -x > gpurun_out/attn_t.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/attn_t.log
timeout 900 python bench.py --attention --no-cpu-baseline --tokens 32768 > gpurun_out/attn_b1.log 2>&1; echo "rc=$?"; grep metric gpurun_out/attn_b1.log > gpurun_out/attn_b1.json; python -c "import json; d=json.load(open('gpurun_out/attn_b1.json')); k=d['kernel_ms_per_layer']; print(round(d['value']), d['ms_per_step'], {x: round(k[x],2) for x in ('gemm1','gemm2','moe')}, d['attention'], d['clocks']['sm_mhz'])"; tail -3 gpurun_out/attn_b1.log
