mkdir -p gpurun_out
timeout 1800 python scripts/sweep.py --gpus 4 --cv 0,0.2 --tokens 32768 --steps 4 --warmup 3 --out gpurun_out/sweep_n4_v3.jsonl > gpurun_out/sweep_n4_v3.log 2>&1; echo "sweep rc=$?"
timeout 1800 python scripts/sweep.py --gpus 4 --cv 0.2 --tokens 32768 --steps 4 --warmup 3 --extra "--engine pull" --out gpurun_out/sweep_n4_v3.jsonl >> gpurun_out/sweep_n4_v3.log 2>&1; echo "sweep pull rc=$?"
timeout 1800 python scripts/sweep.py --gpus 4 --cv 0.2 --tokens 65536 --steps 4 --warmup 3 --extra "--engine hybrid" --out gpurun_out/sweep_n4_v3.jsonl >> gpurun_out/sweep_n4_v3.log 2>&1; echo "sweep hybrid64 rc=$?"
cat gpurun_out/sweep_n4_v3.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'error' in d: print('ERR', d); continue
    print(d['mnt'], d['cv'], round(d['dwdp_tokens_per_s_per_gpu']), round(d['dep_tokens_per_s_per_gpu']), round(d['dwdp_over_dep'],3), round(d['exposed_prefetch_ms_per_layer'],3), d['engine'], round(d['prefetch_gbs'] or 0), d['clocks']['sm_mhz'])"
