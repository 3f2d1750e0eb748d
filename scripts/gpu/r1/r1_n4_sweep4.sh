mkdir -p gpurun_out
for e in pull copy; do timeout 300 python scripts/pull_probe.py --engine $e --plans 2 2>&1 | tail -1 | cut -c1-200; done
timeout 1800 python scripts/sweep.py --gpus 4 --cv 0,0.2 --tokens 32768 --steps 4 --warmup 3 --extra "--engine pull" --out gpurun_out/sweep_n4_v5.jsonl > gpurun_out/sweep_n4_v5.log 2>&1; echo "sweep rc=$?"
cat gpurun_out/sweep_n4_v5.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'error' in d: print('ERR', d); continue
    print(d['mnt'], d['cv'], round(d['dwdp_tokens_per_s_per_gpu']), round(d['dep_tokens_per_s_per_gpu']), round(d['dwdp_over_dep'],3), round(d['exposed_prefetch_ms_per_layer'],3), d['engine'], round(d['prefetch_gbs'] or 0), round(d['step_roofline_frac'],3), d['clocks']['sm_mhz'])"
