# N=4 NVFP4 with the MLA attention window, MNT 32K, CV 0.2.
mkdir -p gpurun_out
timeout 2000 python scripts/sweep.py --gpus 4 --cv 0.2 --tokens 32768 --steps 3 --warmup 3 --extra="--dtype nvfp4 --attention" --out gpurun_out/sweep_n4_fp4_attn.jsonl > gpurun_out/sweep_n4_fp4_attn.log 2>&1; echo "rc=$?"
cat gpurun_out/sweep_n4_fp4_attn.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'error' in d: print('ERR', d); continue
    print(d['mnt'], d['cv'], round(d['dwdp_tokens_per_s_per_gpu']), round(d['dep_tokens_per_s_per_gpu']), round(d['dwdp_over_dep'],3), round(d['exposed_prefetch_ms_per_layer'],3), d['engine'][0], round(d['prefetch_gbs'] or 0), round(d['attention_ms_per_layer'],1), round(d['moe_ms_per_layer'],1))"
