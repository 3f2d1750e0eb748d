# N=2 final build: NVFP4 config-4 points and the bf16 attention-window point.
mkdir -p gpurun_out
timeout 2400 python scripts/sweep.py --gpus 2 --cv 0,0.2 --tokens 32768,65536 --steps 4 --warmup 3 --extra="--dtype nvfp4" --out gpurun_out/sweep_n2_fp4_final.jsonl > gpurun_out/sweep_n2_fp4_final.log 2>&1; echo "sweep rc=$?"
timeout 1800 python scripts/sweep.py --gpus 2 --cv 0.2 --tokens 32768 --steps 3 --warmup 3 --extra=--attention --out gpurun_out/sweep_n2_attn.jsonl > gpurun_out/sweep_n2_attn.log 2>&1; echo "attn rc=$?"
cat gpurun_out/sweep_n2_fp4_final.jsonl gpurun_out/sweep_n2_attn.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'error' in d: print('ERR', d); continue
    print(d['extra'], d['mnt'], d['cv'], round(d['dwdp_tokens_per_s_per_gpu']), round(d['dep_tokens_per_s_per_gpu']), round(d['dwdp_over_dep'],3), round(d['exposed_prefetch_ms_per_layer'],3), d['engine'], round(d['prefetch_gbs'] or 0), d['clocks']['sm_mhz'])"
