# N=4 NVFP4 config-4 points with the round-end build (MNT 32K / 64K, CV 0 / 0.2).
mkdir -p gpurun_out
timeout 2400 python scripts/sweep.py --gpus 4 --cv 0,0.2 --tokens 32768,65536 --steps 4 --warmup 3 --extra="--dtype nvfp4" --out gpurun_out/sweep_n4_fp4_end.jsonl > gpurun_out/sweep_n4_fp4_end.log 2>&1; echo "sweep rc=$?"
cat gpurun_out/sweep_n4_fp4_end.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'error' in d: print('ERR', d); continue
    print(d['mnt'], d['cv'], round(d['dwdp_tokens_per_s_per_gpu']), round(d['dep_tokens_per_s_per_gpu']), round(d['dwdp_over_dep'],3), round(d['exposed_prefetch_ms_per_layer'],3), d['engine'][0], round(d['prefetch_gbs'] or 0), d['clocks']['sm_mhz'])"
