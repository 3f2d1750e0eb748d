# N=4 config-4 sweep at MNT 32K with the MLA attention block in the prefetch window (bf16).
mkdir -p gpurun_out
timeout 3000 python scripts/sweep.py --gpus 4 --cv 0,0.1,0.3 --tokens 32768 --steps 3 --warmup 3 --extra=--attention --out gpurun_out/sweep_n4_attn.jsonl > gpurun_out/sweep_n4_attn.log 2>&1; echo "sweep rc=$?"
cat gpurun_out/sweep_n4_attn.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'error' in d: print('ERR', d); continue
    print(d['mnt'], d['cv'], round(d['dwdp_tokens_per_s_per_gpu']), round(d['dep_tokens_per_s_per_gpu']), round(d['dwdp_over_dep'],3), round(d['exposed_prefetch_ms_per_layer'],3), d['engine'], round(d['prefetch_gbs'] or 0), d['clocks']['sm_mhz'])"
